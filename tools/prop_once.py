"""One config-2 S^2ANTA-prop step repeated (for ncu): python tools/prop_once.py [S] [reps]."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
inp = si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=0, device="cuda")
for i in range(reps):
    santa.decode_prop(inp.q, inp.K, inp.V, inp.seqlens, S, seed=1, offset=i)
torch.cuda.synchronize()
