"""Host cost per decode call (tools only): CPU wall time of K back-to-back calls vs their GPU time,
for the plain binding, the prepared call and a CUDA-graph replay."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01910_b200 as santa  # noqa: E402
import santa_inputs as si  # noqa: E402
inp = si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=0, device="cuda")
geo = santa.make_geometry(inp.q, 8, 32768); ws = santa.workspace(geo, 256, "cuda"); out = torch.empty_like(inp.q)
st = torch.cuda.current_stream()
res = {}
def measure(name, f, K=400):
    for i in range(20): f(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    for i in range(K): f(i)
    e1.record(st); t1 = time.perf_counter(); torch.cuda.synchronize()
    res[name] = {"host_us_per_call": round((t1 - t0) / K * 1e6, 2), "gpu_us_per_call": round(e0.elapsed_time(e1) / K * 1e3, 2)}
measure("binding_decode", lambda i: santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, 256, "stratified", 7, i, out, None, ws, st))
measure("binding_score_phase", lambda i: santa.santa_score_phase(geo, inp.q, inp.K, inp.seqlens, ws, st))
launch = santa.prepare_decode(geo, inp.q, inp.K, inp.V, inp.seqlens, 256, "stratified", 7, out, None, ws, stream=st)
measure("prepared_decode", launch)
print(json.dumps(res))
# the host-buffer step (bench's e2e): pinned [q|k_new|v_new] in, pinned out back
B, H, Hkv, d = 1, 32, 8, 128
qkvh = torch.randn(B * H * d + 2 * B * Hkv * d).to(torch.bfloat16).pin_memory()
qkvd = torch.empty_like(qkvh, device="cuda")
outh = torch.empty(B * H * d, dtype=torch.bfloat16).pin_memory()
measure("host_packed_step", lambda i: santa.santa_decode_step_host_packed(geo, qkvh, qkvd, inp.K, inp.V, inp.seqlens,
                                                                          256, "stratified", 7, i, out, outh, ws,
                                                                          synchronize=False, stream=st))
print(json.dumps(res))
