#!/usr/bin/env python
"""VecEnv step A/B: the bench's env_step leg alone (1M stock envs, fp32 actions resident).
   PRB_LIB_PATH=profiles/ab/libprb_<v>.so python profiles/env_time.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402


class D:
    world = 1

    @staticmethod
    def max(x):
        return x


ctx = pr.Context(0)
m, ind = bench.market_arrays()
market = pr.MarketData(ctx, m["close"], ind)
hbm = json.load(open(os.path.join(bench.ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6536) if hasattr(bench, "ROOT") else 6536
r = bench.env_leg(pr, ctx.lib, ctx, market, pr.StockConfig(), 1 << 20, 6536.0, D())
print(json.dumps({"lib": os.environ.get("PRB_LIB_PATH", "default"), "kernel_us": r["kernel_avg_us"],
                  "frac_hbm": r["frac_hbm"]}))
