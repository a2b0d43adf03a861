"""Probe (tools only): config 3 (batch 32, 32k, S env, default 512) as two half-batch steps whose
sampling overlaps the other half's score pass on a second stream -- score(h1) -> [sample(h1) on a side
stream || score(h2)] -> sample(h2) -- against the single AUTO call.  Two workspaces, batch_offset keeps
the global Philox ids, so the indices equal the single call's."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

S = int(os.environ.get("S", "512"))
B, H, Hkv, d, n = 32, 32, 8, 128, 32768
inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=3, device="cuda")
geo = santa.make_geometry(inp.q, Hkv, n)
ws = santa.workspace(geo, S)
out = torch.empty_like(inp.q)
h = B // 2
halves = []
for i in range(2):
    sl = slice(i * h, (i + 1) * h)
    q, K, V, lens = inp.q[sl], inp.K[sl], inp.V[sl], inp.seqlens[sl]
    g = santa.make_geometry(q, Hkv, n, batch_offset=i * h)
    halves.append((g, q, K, V, lens, santa.workspace(g, S), out[sl]))
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def single(i):
    santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 7, i, out, None, ws,
                                      "two_kernel", main)


def split(i):
    g1, q1, K1, V1, l1, w1, o1 = halves[0]
    g2, q2, K2, V2, l2, w2, o2 = halves[1]
    santa.santa_score_phase(g1, q1, K1, l1, w1, main)
    side.wait_stream(main)
    santa.santa_sample_phase(g1, V1, l1, S, "stratified", 7, i, o1, None, w1, side)
    santa.santa_score_phase(g2, q2, K2, l2, w2, main)
    santa.santa_sample_phase(g2, V2, l2, S, "stratified", 7, i, o2, None, w2, main)
    main.wait_stream(side)


def t(fn, K=10):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for i in range(K):
        fn(i)
    e1.record(main)
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / K * 1e3, 2)


r = {"S": S, "single_two_kernel_us": t(single), "split_overlap_us": t(split)}
o_single = out.clone()
single(0)
torch.cuda.synchronize()
o_single = out.clone()
split(0)
torch.cuda.synchronize()
r["max_abs_diff"] = float((out.float() - o_single.float()).abs().max())
print(json.dumps(r))
