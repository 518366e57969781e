"""Dev: per-CTA timeline of the balanced tcgen05 prefill (TS_PREFILL_TRACE dump)."""
import sys
import numpy as np
h = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64).reshape(-1, 8)
h = h[h[:, 0] > 0]
t0 = h[:, 0].min()
start = (h[:, 0] - t0) / 1e3
end = (h[:, 7] - t0) / 1e3
dur = end - start
print(f"CTAs {len(h)}: start max {start.max():.1f} us; end min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f}; "
      f"duration min {dur.min():.1f} median {np.median(dur):.1f} max {dur.max():.1f}")
order = np.argsort(-end)[:6]
for c in order:
    pe = [(h[c, k] - t0) / 1e3 for k in range(1, 5) if h[c, k] > 0]
    print(f"  cta {c}: start {start[c]:.1f} piece ends {[round(x, 1) for x in pe]} end {end[c]:.1f}")
