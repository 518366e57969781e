"""Dev: summarise a TS_PREFILL_TRACE dump of prefill_tc_kernel (first and last row-block CTAs)."""
import sys
import numpy as np
h = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
for c, name in ((0, "first"), (1, "last")):
    t = h[2048 * c:2048 * (c + 1)]
    if not t[0]:
        continue
    us = lambda x: (x - t[0]) / 1e3
    n = int((t[16:256] > 0).sum())
    print(f"CTA {name}: tiles {n}, cached end {us(t[2]):.1f}, total {us(t[4]):.1f} us")
    nl = int((t[1024:1280] > 0).sum())
    print("  t   S_ready  QK_iss  PV_iss(t)  sm_done   | load l: K_issued V_issued")
    for i in list(range(0, 6)) + list(range(max(6, n - 10), n)):
        print(f"  {i:3d} {us(t[256+i]):8.1f} {us(t[512+i]):7.1f} {us(t[768+i]):8.1f} {us(t[16+i]):9.1f}")
    ii = np.arange(2, min(n, 64))
    print("  t  | QK: start K_landed issued S_ready | PV: start(p_full) V_landed issued | softmax: S_ready xchg P_done pv_waited done")
    for i in list(range(2, 8)) + list(range(min(n, 64) - 4, min(n, 64))):
        f = lambda a: f"{us(t[a + i]):7.2f}"
        print(f"  {i:3d} | {f(512)} {f(576)} {f(640)} {f(256)} | {f(768)} {f(832)} {f(896)} | {f(256)} {f(320)} {f(384)} {f(448)} {f(16)}")
    seg = lambda a, b: np.mean(t[b + ii] - t[a + ii]) / 1e3
    print(f"  softmax per tile: load+exchange {seg(256, 320):.2f}, P {seg(320, 384):.2f}, wait P.V {seg(384, 448):.2f}, "
          f"fold {seg(448, 16):.2f}; S_ready after previous done {np.mean(t[256 + ii] - t[16 + ii - 1]) / 1e3:.2f} us")
    for l in list(range(0, 6)) + list(range(max(6, nl - 26), nl)):
        print(f"    load {l:3d}: K {us(t[1024+l]):8.1f}  V {us(t[1280+l]):8.1f}")
    for nm, a, b in (("K", 1536, 1024), ("V", 1792, 1280)):
        fr, iss = t[a:a + nl], t[b:b + nl]
        print(f"  {nm} loads: free -> issued {np.mean(iss[2:] - fr[2:]) / 1e3:.2f} us (max {np.max(iss[2:] - fr[2:]) / 1e3:.2f})")
