import time, torch, sys, os
sys.path.insert(0, '/root/repo')
import paper_2605_01910_b200 as santa, santa_inputs as si
inp = si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=0, device="cuda")
geo = santa.make_geometry(inp.q, 8, 32768); ws = santa.workspace(geo, 256, "cuda"); out = torch.empty_like(inp.q)
st = torch.cuda.current_stream()
for path in ("step", "two_kernel"):
    for i in range(5): santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, 256, "stratified", 7, i, out, None, ws, path, st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(200): santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, 256, "stratified", 7, i, out, None, ws, path, st)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(path, "host us/call", (t1-t0)/200*1e6, "total us/call", (t2-t0)/200*1e6)
