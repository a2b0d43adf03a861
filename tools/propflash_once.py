"""Config-2 S^2ANTA-prop (S=128) and S^2ANTA-flash (S=2048, tile 256) steps, 3 each (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

inp = si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=0, device="cuda")
for i in range(3):
    santa.decode_prop(inp.q, inp.K, inp.V, inp.seqlens, 128, seed=1, offset=i)
for i in range(3):
    santa.decode_flash(inp.q, inp.K, inp.V, inp.seqlens, 2048, 256, seed=1, offset=i)
torch.cuda.synchronize()
