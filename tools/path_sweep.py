"""Time the two decode paths (single-launch step kernel vs score pass + sampler kernel) over a
batch sweep of the Llama-3.1-8B GQA config (H=32, H_kv=8, d=128, bf16, 32k, S=256 stratified),
back-to-back over rotating caches > 4x L2, CUDA events.  Tools only (prints one JSON line)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402


def main():
    res = {}
    n = 32768
    Ss = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "256").split(",")]
    for B, S in [(int(x), S) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16,32").split(",") for S in Ss]:
        prob = 2 * B * 8 * n * 128 * 2
        NR = max(1, -(-(512 << 20) // prob))
        probs = []
        for r in range(NR):
            inp = si.make_decode_inputs(B, 32, 8, 128, n, dtype="bf16", seed=r, device="cuda")
            geo = santa.make_geometry(inp.q, 8, n)
            probs.append((inp, geo, torch.empty_like(inp.q)))
        ws = santa.workspace(probs[0][1], S, "cuda")
        st = torch.cuda.current_stream()
        row = {}
        for path in ("step", "step_tc", "two_kernel"):
            def f(i):
                inp, geo, out = probs[i % NR]
                santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 7, i, out,
                                                  None, ws, path, st)
            for i in range(5):
                f(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 40 if B <= 4 else 10
            e0.record(st)
            for i in range(K):
                f(i)
            e1.record(st)
            torch.cuda.synchronize()
            row[path] = round(e0.elapsed_time(e1) / K * 1e3, 2)
        row["speedup_step"] = round(row["two_kernel"] / row["step"], 3)
        row["speedup_step_tc"] = round(row["two_kernel"] / row["step_tc"], 3)
        res[f"B{B}_S{S}"] = row
        del probs, ws
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
