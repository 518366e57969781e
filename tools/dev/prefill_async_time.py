"""Dev: host call time and device time of prefill_async vs prefill (device buffers), 512-row chunks at 128K."""
import os, sys, time, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_02886_b200 import selattn as sa
import bench
C, total = 512, 12
eng = sa.Engine(bench.N_CTX + C * (2 * total + 40) + 16, k=bench.K_SEL, n_local=bench.N_LOCAL, n_init=bench.N_INIT,
                chunk_size=C, theta=bench.THETA, num_heads=bench.H, num_kv_heads=bench.H_KV, head_dim=bench.D, block_size=64)
bench.fill_bf16(eng.append_bf16, bench.N_CTX, bench.H_KV * bench.D, torch.device("cuda"), 1234)
q = torch.randn(total, C, bench.H * bench.D, device="cuda")
k = torch.randn(total, C, bench.H_KV * bench.D, device="cuda").to(torch.bfloat16).float()
v = torch.randn(total, C, bench.H_KV * bench.D, device="cuda").to(torch.bfloat16).float()
out = torch.empty(C, bench.H * bench.D, device="cuda")
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
for name, fn in (("sync", lambda i: eng.prefill(q[i], k[i], v[i])), ("async", lambda i: eng.prefill_async(q[i], k[i], v[i], out))):
    host, dev = [], []
    for i in range(total):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        t0 = time.perf_counter()
        fn(i)
        host.append(1e6 * (time.perf_counter() - t0))
        e1.record(st)
        torch.cuda.synchronize()
        dev.append(1e3 * e0.elapsed_time(e1))
    print(name, "host us", [round(x) for x in host], "dev us", [round(x) for x in dev])
# the bench's own timing loop (flush + steps queued behind a device sleep)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for fl in (flush, torch.empty(0, dtype=torch.uint8, device="cuda")):
    us, clocks, launches = bench.timed_steps(st, fl, lambda i: eng.prefill_async(q[i % total], k[i % total], v[i % total], out),
                                             8, 3, 0, 1, sa.launch_count)
    print("timed_steps flush" if fl.numel() else "timed_steps no flush", [round(x) for x in us], launches)
