"""Config-2 two-kernel decode steps (score pass + sample_gather_kernel), 3 reps, for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

inp = si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=0, device="cuda")
for i in range(3):
    santa.decode(inp.q, inp.K, inp.V, inp.seqlens, 256, "stratified", seed=1, offset=i, path="two_kernel")
torch.cuda.synchronize()
