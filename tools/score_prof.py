"""Config-2 (B=1; env B=32: config 3) score pass alone and the two-kernel step (score pass + sampler), back-to-back over 4 rotating
KV caches (> 4x L2), CUDA events (tools only; A/B builds via SANTA_LIB_PATH)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

B = int(os.environ.get("B", "1"))
NR, n, S = max(1, 4 // B), 32768, 256
probs = []
for r in range(NR):
    inp = si.make_decode_inputs(B, 32, 8, 128, n, dtype="bf16", seed=r, device="cuda")
    probs.append((inp, santa.make_geometry(inp.q, 8, n), torch.empty_like(inp.q)))
ws = santa.workspace(probs[0][1], S)
st = torch.cuda.current_stream()


def t(fn, K=int(os.environ.get("K", "400" if B == 1 else "20"))):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K):
        fn(i)
    e1.record(st)
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / K * 1e3, 2)


def score(i):
    inp, geo, _ = probs[i % NR]
    santa.santa_score_phase(geo, inp.q, inp.K, inp.seqlens, ws, st)


def step(i):
    inp, geo, out = probs[i % NR]
    santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 7, i, out, None, ws,
                                      "two_kernel", st)


print(json.dumps({"score_us": t(score), "step_us": t(step), "score_us2": t(score), "step_us2": t(step)}))
