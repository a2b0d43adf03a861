"""Config-2 S^2ANTA-flash timing (tools only): S=2048 / 256 with tiles of 256 keys, back-to-back
over rotating caches > L2; the exact sampler alongside."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402
NR = 4
probs = []
for r in range(NR):
    inp = si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=r, device="cuda")
    probs.append((inp, santa.make_geometry(inp.q, 8, 32768), torch.empty_like(inp.q)))
ws = santa.workspace(probs[0][1], 2048)
st = torch.cuda.current_stream()
def t(fn, K=200):
    for i in range(10): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K): fn(i)
    e1.record(st); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / K * 1e3, 2)
res = {}
for S, tl in ((2048, 256), (256, 256), (2048, 128)):
    def f(i, S=S, tl=tl):
        inp, geo, out = probs[i % NR]
        santa.santa_decode_attention_flash(geo, inp.q, inp.K, inp.V, inp.seqlens, S, tl, 7, i, out, None, ws, st)
    res[f"flash_S{S}_tile{tl}_us"] = t(f)
def g(i):
    inp, geo, out = probs[i % NR]
    santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, 256, "stratified", 7, i, out, None, ws, st)
res["exact_S256_us"] = t(g)
print(json.dumps(res))
