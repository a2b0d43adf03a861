"""Config-2 dense decode (in-repo reference) timing, rotating caches > L2 (tools only)."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402
B = int(os.environ.get("B", "1"))
probs = []
NR = max(1, 4 // B)
for r in range(NR):
    inp = si.make_decode_inputs(B, 32, 8, 128, 32768, dtype="bf16", seed=r, device="cuda")
    probs.append((inp, santa.make_geometry(inp.q, 8, 32768), torch.empty_like(inp.q)))
ws = santa.workspace(probs[0][1], 1)
st = torch.cuda.current_stream()
def f(i):
    inp, geo, out = probs[i % NR]
    santa.santa_dense_reference(geo, inp.q, inp.K, inp.V, inp.seqlens, out, ws, st)
def g(i):
    inp, geo, out = probs[i % NR]
    torch.nn.functional.scaled_dot_product_attention(inp.q.unsqueeze(2), inp.K, inp.V, enable_gqa=True)
def t(fn, K=int(os.environ.get("K", "200"))):
    for i in range(10): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K): fn(i)
    e1.record(st); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / K * 1e3, 2)
print(json.dumps({"dense_us": t(f), "sdpa_us": t(g)}))
