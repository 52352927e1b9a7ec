"""Histogram of QR_PHASE_TIMING lines (build with TT_NVCC_EXTRA=-DQR_PHASE_TIMING):
QRPH m n hasQ ph0..ph4 (clock64 cycles).  Usage: qr_hist.py log"""
import collections
import sys
agg = collections.defaultdict(lambda: [0, 0])
for line in open(sys.argv[1]):
    if not line.startswith("QRPH"):
        continue
    f = line.split()
    m, n = int(f[1]), int(f[2])
    cyc = sum(int(v) for v in f[4:9])
    key = (m // 100 * 100 if m > 1000 else m, n)
    agg[key][0] += 1
    agg[key][1] += cyc
tot = sum(v[1] for v in agg.values())
print(f"{sum(v[0] for v in agg.values())} QRs, {tot / 1.965e6:.1f} ms at 1965 MHz (sum over launches)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"m {k[0]:7d} n {k[1]:4d}: {v[0]:6d} x {v[1] / v[0] / 1.965e3:8.1f} us = {v[1] / 1.965e6:8.1f} ms")
