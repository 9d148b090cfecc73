#!/usr/bin/env python
"""Print the clock64 phase trace of CTA 0 / thread 0 of the stock tcgen05 rollout
(PRB_TC_TRACE=<file> python profiles/drive.py collect ...): per step, the
cycles spent in each phase (16 marks per step)."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
names = ["X build", "L1 mma", "epi a1", "L2a mma", "epi c1", "L2c mma", "epi a2", "L3a issue", "critic head", "L3a wait",
         "obs rows", "sample", "act rows", "env step", "writes", "->next"]
steps = [h for h in range(2, 30) if t[16 * h + 15] > 0][:6]
acc = np.zeros(16)
for h in steps:
    m = t[16 * h:16 * h + 17]
    acc += np.diff(m)
acc /= len(steps)
tot = acc.sum()
for n, v in zip(names, acc):
    print(f"  {n:10s} {v:8.0f} clk  {100 * v / tot:5.1f}%")
print(f"  step total {tot:8.0f} clk")
