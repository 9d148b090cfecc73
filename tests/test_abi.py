"""CPU-only checks of the product C ABI: the library loads, exports every
symbol include/prb.h declares, and its host-side logic (seeds, synthetic
market, indicators, artifact_init) matches the oracle / reference exactly."""
import ctypes as C
import os
import re

import numpy as np

from oracle_bind import derive_seed as orc_derive, indicators as orc_indicators, ptr, SZ

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "prb.h")).read()
    return sorted(set(re.findall(r"PRB_API\s+[^;(]*?\b(prb_\w+)\s*\(", txt)))


def test_header_symbols_exported(prb):
    names = declared_symbols()
    assert len(names) > 50
    cdll = C.CDLL(prb.path)
    missing = [n for n in names if not hasattr(cdll, n)]
    assert not missing, missing


def test_python_binding_covers_header(prb):
    from paper_2112_05923_b200._lib import SIGNATURES
    assert set(declared_symbols()) == set(SIGNATURES)


def test_no_cpu_fallback_symbols(prb):
    # the product library must not carry the checker: no oracle/ref entry points linked in
    cdll = C.CDLL(prb.path)
    for n in ("orc_stock_env_step", "ref_stock_env_step", "orc_ppo_update"):
        assert not hasattr(cdll, n)


def test_derive_seed_matches_oracle(orc):
    from paper_2112_05923_b200 import podracer as pr
    rng = np.random.default_rng(1)
    for _ in range(100):
        base = int(rng.integers(0, 2**63))
        tags = [int(x) for x in rng.integers(0, 2**32, size=int(rng.integers(0, 4)))]
        assert pr.derive_seed(base, *tags) == orc_derive(orc, base, *tags)


def test_indicators_match_oracle(orc):
    from paper_2112_05923_b200 import podracer as pr
    m = pr.synthetic_market(6, 400, seed=9)
    got = pr.compute_indicators(m["high"], m["low"], m["close"])
    exp = orc_indicators(orc, m["high"], m["low"], m["close"])
    assert np.array_equal(got, exp)


def test_indicators_reject_short_series():
    from paper_2112_05923_b200 import podracer as pr
    m = pr.synthetic_market(2, 34, seed=1)
    try:
        pr.compute_indicators(m["high"], m["low"], m["close"])
    except pr.DataError:
        return
    raise AssertionError("expected DataError (market.hpp:374-378)")


def test_synthetic_market_shape_and_determinism():
    from paper_2112_05923_b200 import podracer as pr
    a = pr.synthetic_market(30, 2048, seed=2112)
    b = pr.synthetic_market(30, 2048, seed=2112)
    assert np.array_equal(a["close"], b["close"])
    c = a["close"]
    assert np.all((c[:, 0] >= 10) & (c[:, 0] <= 200))
    lr = np.log(c[:, 1:] / c[:, :-1])
    assert abs(lr.std() - 1e-3) < 5e-5 and np.allclose(a["high"], 1.001 * c) and np.all(a["volume"] == 1000.0)


def test_artifact_init_matches_reference(ref):
    from paper_2112_05923_b200 import podracer as pr
    for S, A, hid, seed in [(181, 30, (64, 64), 7), (6, 2, (256, 256, 256), 3), (3, 1, (8,), 1)]:
        got = pr.artifact_init(S, A, seed, hid)
        h = np.array(hid, dtype=np.uint64)
        n = ref.ref_artifact_init(S, A, seed, 1e-3, ptr(h, SZ), len(hid), None)
        exp = np.zeros(n)
        ref.ref_artifact_init(S, A, seed, 1e-3, ptr(h, SZ), len(hid), ptr(exp))
        assert np.array_equal(got, exp)
    assert pr.artifact_init(181, 30, 7).size == 33661  # P = 33,661
    assert pr.artifact_init(6, 2, 7, (256, 256, 256)).size == 267525
