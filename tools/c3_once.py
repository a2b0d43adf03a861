"""Run the config-3 decode (batch 32, 32k, S=256, AUTO path = tensor-core step kernel) a few times
(for ncu captures of the large-batch kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

B, H, Hkv, d, n, S = 32, 32, 8, 128, 32768, 256
inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=77, device="cuda")
geo = santa.make_geometry(inp.q, Hkv, n)
ws = santa.workspace(geo, S, "cuda")
out = torch.empty_like(inp.q)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 7, i, out, None, ws)
torch.cuda.synchronize()
print("ok")
