import torch, time, statistics
h = torch.zeros(6144, dtype=torch.float32).pin_memory()
d = torch.zeros(6144, dtype=torch.float32, device="cuda")
x = torch.zeros(16, device="cuda")
s = torch.cuda.Stream()
res = []
with torch.cuda.stream(s):
    for i in range(200):
        e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda._sleep(20000)
        e0.record(s); d.copy_(h, non_blocking=True); e1.record(s); x.add_(1); e2.record(s)
        s.synchronize()
        res.append((e0.elapsed_time(e1) * 1000, e1.elapsed_time(e2) * 1000))
print("H2D 24KB device time us: median", statistics.median(r[0] for r in res[20:]), " tiny kernel after:", statistics.median(r[1] for r in res[20:]))
res = []
with torch.cuda.stream(s):
    for i in range(200):
        e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda._sleep(20000)
        e0.record(s); x.add_(1); e1.record(s); x.add_(1); e2.record(s)
        s.synchronize()
        res.append((e0.elapsed_time(e1) * 1000, e1.elapsed_time(e2) * 1000))
print("tiny kernel device time us: median", statistics.median(r[0] for r in res[20:]), statistics.median(r[1] for r in res[20:]))
dd = torch.zeros(4096, device="cuda")
res = []
with torch.cuda.stream(s):
    for i in range(200):
        e0, e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda._sleep(20000)
        e0.record(s); h[:4096].copy_(dd, non_blocking=True); e1.record(s)
        s.synchronize()
        res.append(e0.elapsed_time(e1) * 1000)
print("D2H 16KB device time us: median", statistics.median(res[20:]))
