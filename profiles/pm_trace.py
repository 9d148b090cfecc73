#!/usr/bin/env python
"""Print the clock64 phase trace of CTA 0 of the PointMass tcgen05 rollout
(PRB_PM_TRACE=<file> python profiles/drive.py pm ...).  Per step:
  actor : X-ready, then (L1..L3) dfull-recv / epi-done, L4 recv, env-done  (9)
  critic: (L1..L3) dfull-recv / epi-done, L4 recv, value-done             (8)
  mma   : per op A1 C4(prev) C1 A2 C2 A3 C3 A4: ready-recv, commit           (16)"""
import sys

import numpy as np

L = 512
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(4, L).astype(np.int64)
steps = range(int(sys.argv[2]) if len(sys.argv) > 2 else 2, int(sys.argv[3]) if len(sys.argv) > 3 else 5)
for h in steps:
    a, c, m = t[0, 9 * h:9 * h + 9], t[1, 8 * h:8 * h + 8], t[2, 16 * h - 2:16 * h + 14]
    t0 = a[0]
    print(f"step {h}: period {t[0, 9 * (h + 1)] - t0} clk")
    print("  actor :", " ".join(f"{x - t0:6d}" for x in a))
    print("  critic:", " ".join(f"{x - t0:6d}" for x in c))
    print("  mma   :", " ".join(f"{x - t0:6d}" for x in m))
    if h < 8:
        print("  mma waited for chunks (cumulative):", t[3, h])
        if t[3, 16 + h]:
            print("  ... of which waiting for the peer CTA's half (cumulative):", t[3, 16 + h])
