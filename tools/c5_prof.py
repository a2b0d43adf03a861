"""Config 5 (batch 16, 32k, Bernoulli mean-group stratified B=8 + S=256) -- time the Bernoulli decode
step and the standalone score stage (tools only; used under ncu too)."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402
B, H, Hkv, d, n, S = 16, 32, 8, 128, 32768, 256
inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=5, workload="lognormal", feature_major=True,
                            device="cuda")
geo = santa.make_geometry(inp.q, Hkv, n)
ws = santa.workspace(geo, S)
out = torch.empty_like(inp.q)
sc = torch.empty(B, H, n, device="cuda")
st = torch.cuda.current_stream()
def t(fn, K=int(os.environ.get("K", "20"))):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K): fn(i)
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3
r = {"decode_bernoulli_us": t(lambda i: santa.santa_decode_attention_bernoulli(geo, inp.q, inp.Kt, inp.V, inp.seqlens, 8, 1, 1, S, "stratified", 13, i, out, None, ws)),
     "bernoulli_scores_us": t(lambda i: santa.santa_bernoulli_scores(geo, inp.q, inp.Kt, inp.seqlens, 8, 1, 1, 13, i, sc, None, ws))}
print(json.dumps(r))
