"""Run the config-5 decode (Bernoulli + S2ANTA, batch 16, 32k) a few times (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

Bt, H, Hkv, d, n, S, nB = 16, 32, 8, 128, 32768, 256, 8
inp = si.make_decode_inputs(Bt, H, Hkv, d, n, dtype="bf16", workload="lognormal", seed=500, feature_major=True,
                            device="cuda")
geo = santa.make_geometry(inp.q, Hkv, n)
ws = santa.workspace(geo, S, "cuda")
out = torch.empty_like(inp.q)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    santa.santa_decode_attention_bernoulli(geo, inp.q, inp.Kt, inp.V, inp.seqlens, nB, 1, 1, S, "stratified", 7, i,
                                           out, None, ws)
torch.cuda.synchronize()
print("ok")
