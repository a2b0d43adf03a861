"""Per-phase timeline of the cluster sampler (sample_gather_kernel) at config 5 (batch 16, 32k,
Bernoulli mean-group B=8 + S=256) or config 3 (env CFG=3: batch 32, exact score pass, path two_kernel):
the library's sampler writes globaltimer stamps of thread 0 of every head's CTA when
SANTA_SAMPLE_TRACE holds a device buffer address (tools only).  Prints the median / p90 time of each
phase relative to that CTA's start and to the earliest start.  Phases: 0 start, 1 thresholds,
2 after griddepcontrol.wait (score pass done), 3 chunk stats loaded + max, 4 fp64 CDF built,
5 chunk of every sample found, 8 every J known, 9 V rows added, 6 half-warp partials in smem, 7 end."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CFG = int(os.environ.get("CFG", "5"))
R = int(os.environ.get("R", "2"))  # CFG=4: rank 0's phase 2 of a 512k sequence sharded over R ranks
B, H, Hkv, d, n, S = (16 if CFG == 5 else 32), 32, 8, 128, 32768, int(os.environ.get("S", "256"))
if CFG == 4:
    B, n, S = 1, 524288 // R, int(os.environ.get("S", "1024"))
trace = torch.zeros(B * H * 16, dtype=torch.int64, device="cuda")
os.environ["SANTA_SAMPLE_TRACE"] = hex(trace.data_ptr())
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402

if CFG == 5:
    inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=5, workload="lognormal", feature_major=True,
                                device="cuda")
elif CFG == 4:
    from paper_2605_01910_b200 import sharding
    inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=5, device="cuda")
    be = sharding.CudaBackend()
    st4 = be.stats(inp.q, inp.K, inp.seqlens, Hkv, S)
    stats_all = st4.unsqueeze(0).repeat(R, 1, 1, 1).contiguous()
    off = torch.zeros(1, dtype=torch.int32, device="cuda")
else:
    inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=5, device="cuda")
geo = santa.make_geometry(inp.q, Hkv, n)
ws = santa.workspace(geo, S)
out = torch.empty_like(inp.q)


def run(i):
    if CFG == 4:
        be.sample_gather(stats_all, 0, R, off, inp.V, inp.seqlens, S, "stratified", 13, i)
    elif CFG == 5:
        santa.santa_decode_attention_bernoulli(geo, inp.q, inp.Kt, inp.V, inp.seqlens, 8, 1, 1, S, "stratified", 13,
                                               i, out, None, ws)
    else:
        santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 13, i, out, None,
                                          ws, "two_kernel")


res = {}
for rep in range(5):
    trace.zero_()
    run(rep)
    torch.cuda.synchronize()
    t = trace.view(B * H, 16).cpu().double()
    t0 = t[:, 0]
    base = t0.min()
    for ph in (1, 2, 3, 4, 5, 8, 9, 6, 7):
        col = t[:, ph]
        ok = col > 0
        rel = (col[ok] - t0[ok]) / 1e3
        ab = (col[ok] - base) / 1e3
        res.setdefault(ph, []).append((rel.median().item(), rel.quantile(0.9).item(), ab.median().item(),
                                       ab.max().item()))
    res.setdefault("start_spread_us", []).append(((t0 - base) / 1e3).max().item())
out_ = {}
for k, v in res.items():
    v = v[1:]  # drop the first (cold) repetition
    if k == "start_spread_us":
        out_[k] = round(sorted(v)[len(v) // 2], 2)
    else:
        out_[f"phase{k}"] = {"rel_med_us": round(sorted(x[0] for x in v)[len(v) // 2], 2),
                             "rel_p90_us": round(sorted(x[1] for x in v)[len(v) // 2], 2),
                             "abs_med_us": round(sorted(x[2] for x in v)[len(v) // 2], 2),
                             "abs_max_us": round(sorted(x[3] for x in v)[len(v) // 2], 2)}
print(json.dumps({"cfg": CFG, "S": S, **out_}))
