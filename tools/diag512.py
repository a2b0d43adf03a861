import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2605_01910_b200 as santa
from paper_2605_01910_b200 import sharding
import santa_inputs as si
from oracle import santa_oracle as o
from gpu_helpers import gpu_decode
n, S = 524288, 1024
inp = si.make_decode_inputs(1, 32, 8, 128, n, dtype="bf16", seed=43, device="cuda")
out_f, idx_f = gpu_decode(inp, S, "stratified", seed=7, offset=3)
be = sharding.CudaBackend()
sl = torch.tensor([n], dtype=torch.int32, device="cuda")
st = be.stats(inp.q, inp.K, sl, 8, S)
part, idx_s = be.sample_gather(st.unsqueeze(0), 0, 1, torch.zeros(1, dtype=torch.int32, device="cuda"), inp.V, sl, S, "stratified", 7, 3, return_idx=True)
torch.cuda.synchronize()
print("fast vs old differ:", (idx_f != idx_s).sum().item(), "of", idx_f.numel())
for kv in range(8):
    sub_q = si.as_bits(inp.q[:, 4*kv:4*kv+4]); sub_K = si.as_bits(inp.K[:, kv:kv+1]); sub_V = si.as_bits(inp.V[:, kv:kv+1])
    _, idx_o, det = o.santa_decode(sub_q, sub_K, sub_V, [n], S, "stratified", 7, 3, head_offset=4*kv, return_details=True)
    for name, ig in (("fast", idx_f), ("old", idx_s)):
        g = ig[:, 4*kv:4*kv+4].cpu().numpy().astype(np.int64)
        tot, mis, ex, fails = o.index_mismatch_report(det["F"], det["T"], idx_o, g)
        print(kv, name, "mismatch", mis, "exempt", ex, "FAIL", len(fails), fails[:2])
