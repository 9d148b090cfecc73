"""Generate tests/golden/ref_golden_r2.npz from the REFERENCE ITSELF (round-2 additions).

Same recipe as make_golden.py: every vector comes from oracle/_ref/libpodracer_ref_exact.so,
i.e. the unmodified reference headers compiled behind oracle/ref_shim.cpp.  Kept in a separate
file so ref_golden.npz stays byte-identical.

Run from the repo root after build():  python tests/golden/make_golden_r2.py
Reference calls used:
  leaderboard_update + Leaderboard::refresh_stats   tournament.hpp:66-119
  encode_checkpoint(artifact_to_tensors(...))       checkpoint.hpp:122-245
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bind import load_ref, ptr, I64, SZ, U8  # noqa: E402

LBS_SHAPE = (5, 2, (4,))  # S, A, hidden: P = 65


def param_count(S, A, hidden):
    dims = [S, *hidden]
    actor = sum((i + 1) * o for i, o in zip(dims, dims[1:] + [A]))
    critic = sum((i + 1) * o for i, o in zip(dims, dims[1:] + [1]))
    return actor + A + critic


def leaderboard_stats(ref, cand, scores, ids, cap, S, A, hidden):
    hid = np.array(hidden, dtype=np.uint64)
    P = cand.shape[1]
    oi = np.full(cap, -1, np.int64); osz = C.c_size_t(); mean = np.zeros(P); var = np.zeros(P)
    assert ref.ref_leaderboard_stats(ptr(np.ascontiguousarray(cand)), ptr(scores), ptr(ids, I64), len(scores), cap,
                                     S, A, ptr(hid, SZ), len(hidden), ptr(oi, I64), C.byref(osz), ptr(mean),
                                     ptr(var)) == 0
    return oi[:osz.value], mean, var


def main():
    ref = load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libpodracer_ref_exact.so missing: build() in a container with /root/reference")
    out = {}
    rng = np.random.default_rng(2026)

    # leaderboard population stats: 8 sequences of 12 candidates (fp32-representable params, so the
    # device's fp32 parameter blobs hold exactly the reference's values), capacity 1..6, ties
    S, A, hidden = LBS_SHAPE
    P = param_count(S, A, hidden)
    cands, scores, caps, boards, means, vars_ = [], [], [], [], [], []
    for trial in range(8):
        cap = int(1 + trial % 6)
        c = rng.normal(scale=0.5, size=(12, P)).astype(np.float32).astype(np.float64)
        s = rng.integers(0, 5, 12).astype(np.float64) if trial % 2 else rng.uniform(-1, 1, 12)
        ids = np.arange(12, dtype=np.int64)
        b, m, v = leaderboard_stats(ref, c, s, ids, cap, S, A, hidden)
        cands.append(c); scores.append(s); caps.append(cap)
        boards.append(np.concatenate([b, np.full(6 - len(b), -1)]).astype(np.int64)); means.append(m); vars_.append(v)
    out.update(lbs_cand=np.array(cands, np.float32), lbs_scores=np.array(scores), lbs_cap=np.array(caps),
               lbs_board=np.array(boards), lbs_mean=np.array(means), lbs_var=np.array(vars_),
               lbs_shape=np.array([S, A, *hidden], np.int64))

    # PODRCKPT v1 bytes written by the reference (checkpoint.hpp: encode_checkpoint(artifact_to_tensors))
    # for a small artifact with Adam state, lineage, a custom algo tag and meta; and without meta
    S2, A2, hid2 = 4, 2, np.array([3], dtype=np.uint64)
    P2 = param_count(S2, A2, (3,))
    ck_flat = rng.normal(size=P2); ck_m = rng.normal(size=P2) * 1e-2; ck_v = rng.uniform(0, 1e-3, P2)
    hyper = np.array([0.9, 0.999, 1e-8, 3e-4])
    meta = np.array([12.5, 4096.0, -0.75])
    blobs = []
    for with_meta, tag, parent, mseed in ((True, b"ppo", 7, 2**63 + 12345), (False, b"ppo-b200", -1, 99)):
        n = ref.ref_checkpoint_encode(ptr(ck_flat), ptr(ck_m), ptr(ck_v), 17, ptr(hyper), S2, A2, ptr(hid2, SZ), 1,
                                      parent, mseed, tag, ptr(meta) if with_meta else None, None)
        buf = np.zeros(n, np.uint8)
        ref.ref_checkpoint_encode(ptr(ck_flat), ptr(ck_m), ptr(ck_v), 17, ptr(hyper), S2, A2, ptr(hid2, SZ), 1,
                                  parent, mseed, tag, ptr(meta) if with_meta else None, ptr(buf, U8))
        blobs.append(buf)
    out.update(ck_flat=ck_flat, ck_m=ck_m, ck_v=ck_v, ck_hyper=hyper, ck_meta=meta, ck_bytes_meta=blobs[0],
               ck_bytes_nometa=blobs[1], ck_shape=np.array([S2, A2, 3], np.int64))

    path = os.path.join(HERE, "ref_golden_r2.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
