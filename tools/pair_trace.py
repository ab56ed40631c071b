"""Print the per-tile timeline of cluster 0 of the pair kernel from gpurun_out/pair_trace.bin (experiment build,
PPCA_TRACE=k).  Events (clock64 of each CTA's SM): 0 P1 start (TMEM free), 1 P1 issued, 2/3 warp 0 drain/exchange
done, 4/5 warp 2 drain/exchange done, 6 P2 start (Y landed), 7 P2+S issued, 8/9 A-stream first/last chunk issued."""
import sys
import numpy as np

T, E = 128, 12
raw = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/pair_trace.bin", dtype=np.int64)
a = raw[: 2 * T * E].reshape(2, T, E)
g = raw[2 * T * E:].reshape(-1, 2)
g = g[g[:, 0] > 0]
g0 = g[:, 0].min()
st, en = (g[:, 0] - g0) / 1e3, (g[:, 1] - g0) / 1e3
print(f"all CTAs ({len(g)}): product-1 start {st.min():.1f}..{st.max():.1f} us, end min {en.min():.1f} median {np.median(en):.1f} max {en.max():.1f} us")
print("  end-time deciles:", " ".join(f"{v:.0f}" for v in np.percentile(en, np.arange(0, 101, 10))))
for h in range(2):
    b = a[h]
    n = int((b[:, 0] > 0).sum())
    t0 = b[0, 0]
    g = b[:n, 10]
    ghz = (b[n - 1, 0] - b[0, 0]) / max(g[n - 1] - g[0], 1)
    print(f"CTA {h}: SM clock {ghz:.3f} GHz (clock64 / globaltimer over the traced tiles)")
    us = (b[:n] - t0) / ghz / 1e3
    print(f"CTA {h}: {n} tiles, period {np.median(np.diff(us[:, 0])):.2f} us")
    print(" tile  P1start P1issued  w0tfull w0exch  w2tfull w2exch  P2start P2issued  A0    A7")
    for i in list(range(0, 6)) + list(range(n // 2, n // 2 + 4)):
        print(f"{i:5d} " + " ".join(f"{v:7.2f}" for v in us[i, :10]))
    d = np.diff(us, axis=0)
    print(" median gaps: P1 issue dur %.2f | tfull->exch w0 %.2f w2 %.2f | P1issued->w0tfull %.2f | w0exch->P2start %.2f | P2 dur %.2f" % (
        np.median(us[:, 1] - us[:, 0]), np.median(us[:, 3] - us[:, 2]), np.median(us[:, 5] - us[:, 4]),
        np.median(us[:, 2] - us[:, 1]), np.median(us[:, 6] - np.maximum(us[:, 3], us[:, 5])), np.median(us[:, 7] - us[:, 6])))
