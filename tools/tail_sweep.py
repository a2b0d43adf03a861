"""Config-2 tail tuning (tools only): two-kernel step time and the sample phase alone for a list of
sampler cluster sizes (SANTA_FAST_CS), back-to-back over rotating caches > 4x L2, CUDA events.
Usage: python tools/tail_sweep.py [B] [S] [cs,cs,...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402


def timeit(f, K=200, W=20):
    st = torch.cuda.current_stream()
    for i in range(W):
        f(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K):
        f(i)
    e1.record(st)
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / K * 1e3, 2)


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    css = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4,8").split(",")]
    n = 32768
    prob = 2 * B * 8 * n * 128 * 2
    NR = max(1, -(-(512 << 20) // prob))
    probs = []
    for r in range(NR):
        inp = si.make_decode_inputs(B, 32, 8, 128, n, dtype="bf16", seed=r, device="cuda")
        geo = santa.make_geometry(inp.q, 8, n)
        probs.append((inp, geo, torch.empty_like(inp.q)))
    wss = [santa.workspace(probs[0][1], S, "cuda") for _ in range(NR)]
    st = torch.cuda.current_stream()
    res = {}
    for cs in css:
        os.environ["SANTA_FAST_CS"] = str(cs)

        def step(i):
            inp, geo, out = probs[i % NR]
            santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 7, i, out,
                                              None, wss[0], "two_kernel", st)
        for r in range(NR):  # score phase into each workspace once
            inp, geo, out = probs[r]
            santa.santa_score_phase(geo, inp.q, inp.K, inp.seqlens, wss[r], st)

        def sample(i):
            inp, geo, out = probs[i % NR]
            santa.santa_sample_phase(geo, inp.V, inp.seqlens, S, "stratified", 7, i, out, None, wss[i % NR], st)
        res[cs] = {"step_us": timeit(step), "sample_phase_us": timeit(sample)}
    def score(i):
        inp, geo, out = probs[i % NR]
        santa.santa_score_phase(geo, inp.q, inp.K, inp.seqlens, wss[0], st)
    res["score_phase_us"] = timeit(score)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
