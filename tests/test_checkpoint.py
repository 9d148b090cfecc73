"""PODRCKPT v1 checkpoints (checkpoint.hpp:16-317) through the product library's host codec
(prb_checkpoint_encode_host / _decode_host; CPU only).

  * bytes written by the REFERENCE (tests/golden/ref_golden_r2.npz, make_golden_r2.py) decode to
    the exact values, and re-encoding the same artifact gives the identical byte image;
  * against the reference build directly (oracle/_ref) for random artifacts, when it is built;
  * error classes in the reference's order: CRC (CorruptionError) before magic (FormatError) and
    version (VersionError); truncation / trailing bytes are corruption.
"""
import ctypes as C
import os
import struct
import zlib

import numpy as np
import pytest

from oracle_bind import ptr, SZ, U8

GOLDEN_R2 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden_r2.npz")


def encode_host(prb, S, A, hid, flat, m, v, t, hyper, parent, mseed, tag, meta):
    h = np.array(hid, dtype=np.uint64)
    size = C.c_size_t()
    args = [S, A, h.ctypes.data_as(C.POINTER(C.c_size_t)), len(hid), ptr(flat), ptr(m), ptr(v), t, ptr(hyper), parent,
            mseed, tag, ptr(meta) if meta is not None else None]
    prb.prb_checkpoint_encode_host(*args, None, 0, C.byref(size))
    out = np.zeros(size.value, np.uint8)
    prb.prb_checkpoint_encode_host(*args, out.ctypes.data_as(C.POINTER(C.c_uint8)), out.size, C.byref(size))
    return out


def decode_host(prb, data, S, A, hid, P):
    h = np.array(hid, dtype=np.uint64)
    flat, m, v, hyper, meta = np.zeros(P), np.zeros(P), np.zeros(P), np.zeros(4), np.zeros(3)
    t, parent, seed, has = C.c_int64(), C.c_int64(), C.c_uint64(), C.c_int()
    tag = C.create_string_buffer(64)
    b = np.frombuffer(bytes(data), dtype=np.uint8).copy()
    prb.prb_checkpoint_decode_host(b.ctypes.data_as(C.POINTER(C.c_uint8)), b.size, S, A,
                                   h.ctypes.data_as(C.POINTER(C.c_size_t)), len(hid), ptr(flat), ptr(m), ptr(v),
                                   C.byref(t), ptr(hyper), C.byref(parent), C.byref(seed), tag, 64, ptr(meta),
                                   C.byref(has))
    return dict(flat=flat, m=m, v=v, t=t.value, hyper=hyper, parent=parent.value, seed=seed.value,
                tag=tag.value.decode(), meta=meta if has.value else None)


def test_reference_bytes_decode_and_reencode(prb):
    g = np.load(GOLDEN_R2)
    S, A, h = (int(x) for x in g["ck_shape"])
    P = g["ck_flat"].size
    for key, tag, parent, mseed, meta in (("ck_bytes_meta", "ppo", 7, 2**63 + 12345, g["ck_meta"]),
                                         ("ck_bytes_nometa", "ppo-b200", -1, 99, None)):
        d = decode_host(prb, g[key].tobytes(), S, A, [h], P)
        assert np.array_equal(d["flat"], g["ck_flat"]) and np.array_equal(d["m"], g["ck_m"])
        assert np.array_equal(d["v"], g["ck_v"]) and d["t"] == 17 and np.array_equal(d["hyper"], g["ck_hyper"])
        assert (d["parent"], d["seed"], d["tag"]) == (parent, mseed, tag)
        assert (d["meta"] is None) == (meta is None) and (meta is None or np.array_equal(d["meta"], meta))
        again = encode_host(prb, S, A, [h], g["ck_flat"], g["ck_m"], g["ck_v"], 17, g["ck_hyper"], parent, mseed,
                            tag.encode(), meta)
        assert again.tobytes() == g[key].tobytes()


def test_encode_matches_reference_build(prb, ref):
    rng = np.random.default_rng(9)
    for S, A, hid in ((181, 30, (64, 64)), (6, 2, (8,)), (3, 1, (4, 5, 6))):
        P = sum((i + 1) * o for i, o in zip([S, *hid], [*hid, A])) + A + sum((i + 1) * o for i, o in zip([S, *hid], [*hid, 1]))
        flat, m, v = rng.normal(size=P), rng.normal(size=P) * 1e-3, rng.uniform(0, 1e-4, P)
        hyper = np.array([0.8, 0.99, 1e-7, 1e-3])
        h = np.array(hid, dtype=np.uint64)
        n = ref.ref_checkpoint_encode(ptr(flat), ptr(m), ptr(v), 5, ptr(hyper), S, A, ptr(h, SZ), len(hid), 3, 42,
                                      b"ppo", None, None)
        want = np.zeros(n, np.uint8)
        ref.ref_checkpoint_encode(ptr(flat), ptr(m), ptr(v), 5, ptr(hyper), S, A, ptr(h, SZ), len(hid), 3, 42,
                                  b"ppo", None, ptr(want, U8))
        got = encode_host(prb, S, A, list(hid), flat, m, v, 5, hyper, 3, 42, b"ppo", None)
        assert got.tobytes() == want.tobytes()
        # the reference decodes ours
        f2, m2, v2 = np.zeros(P), np.zeros(P), np.zeros(P)
        t2, p2, s2 = C.c_int64(), C.c_int64(), C.c_uint64()
        assert ref.ref_checkpoint_decode(ptr(got, U8), got.size, ptr(f2), ptr(m2), ptr(v2), C.byref(t2), C.byref(p2),
                                         C.byref(s2)) == 0
        assert np.array_equal(f2, flat) and np.array_equal(m2, m) and t2.value == 5 and s2.value == 42


def _with_crc(body: bytes) -> bytes:
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def test_error_classes(prb):
    from paper_2112_05923_b200 import _lib
    g = np.load(GOLDEN_R2)
    S, A, h = (int(x) for x in g["ck_shape"])
    P = g["ck_flat"].size
    good = g["ck_bytes_meta"].tobytes()
    assert zlib.crc32(good[:-4]) & 0xFFFFFFFF == struct.unpack("<I", good[-4:])[0]  # CRC-32 IEEE, as zlib's
    bad_crc = bytearray(good)
    bad_crc[40] ^= 0x01
    with pytest.raises(_lib.CorruptionError):
        decode_host(prb, bad_crc, S, A, [h], P)
    with pytest.raises(_lib.FormatError):
        decode_host(prb, _with_crc(b"NOTACKPT" + good[8:-4]), S, A, [h], P)
    with pytest.raises(_lib.VersionError):
        decode_host(prb, _with_crc(good[:8] + struct.pack("<I", 2) + good[12:-4]), S, A, [h], P)
    with pytest.raises(_lib.CorruptionError):
        decode_host(prb, _with_crc(good[:-20]), S, A, [h], P)  # truncated tensor payload
    with pytest.raises(_lib.CorruptionError):
        decode_host(prb, _with_crc(good[:-4] + bytes(8)), S, A, [h], P)  # trailing bytes
    with pytest.raises(_lib.CorruptionError):
        decode_host(prb, good[:10], S, A, [h], P)  # too short
    with pytest.raises(_lib.DimensionError):
        decode_host(prb, good, S + 1, A, [h], P + 3)  # another agent shape
