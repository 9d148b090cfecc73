#!/usr/bin/env python
"""Per-CTA placement and span of the stock tcgen05 rollout (the PRB_TC_TRACE file of a
-DPRB_DEBUG_KNOBS build: after the 512 clock64 marks of CTA 0, (smid, start, end) globaltimer
stamps per CTA).  Prints CTAs per SM, the spread of start / end times and per-SM load.
    python profiles/tc_cta_span.py <trace.bin> <num_envs>"""
import sys
from collections import Counter

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
n = (int(sys.argv[2]) + 127) // 128
x = t[512:512 + 3 * n].reshape(n, 3)
sm, st, en = x[:, 0], x[:, 1], x[:, 2]
t0 = st.min()
st, en = (st - t0) / 1e3, (en - t0) / 1e3
c = Counter(sm.tolist())
print(f"{n} CTAs on {len(c)} SMs; CTAs per SM histogram: {sorted(Counter(c.values()).items())}")
print(f"start us: min {st.min():.1f} median {np.median(st):.1f} max {st.max():.1f}")
print(f"end   us: min {en.min():.1f} median {np.median(en):.1f} max {en.max():.1f}")
dur = en - st
for k in sorted(set(c.values())):
    sel = np.array([c[s] == k for s in sm])
    print(f"  CTAs on SMs holding {k}: duration median {np.median(dur[sel]):.1f} us, max {dur[sel].max():.1f}")
