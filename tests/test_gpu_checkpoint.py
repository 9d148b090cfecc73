"""GPU: the device-resident generator's fresh init and checkpoints of device agents.

  * prb_agent_init_device == artifact_init (artifact.hpp:91-105, nn.hpp:40-54) rounded to fp32, bit
    for bit, for the stock 64x64 and the PointMass 3x256 nets (the reference's mt19937_64 streams
    and uniform_real_distribution drawn on the device).
  * an agent's PODRCKPT bytes equal the host codec's encoding of its (fp32 -> f64) state, which the
    CPU suite pins to the reference's own bytes; decode into a fresh agent restores params, m, v,
    t and hyper-parameters exactly; save / load through a file; a reference-written checkpoint
    loads (values rounded to fp32 once).
"""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN_R2 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden_r2.npz")


@pytest.fixture(scope="module")
def pr():
    from paper_2112_05923_b200 import podracer
    return podracer


@pytest.fixture(scope="module")
def ctx(pr):
    return pr.Context(0)


@pytest.mark.parametrize("S,A,hid,seed", [(181, 30, (64, 64), 7), (6, 2, (256, 256, 256), 11), (5, 3, (4,), 2**63 + 5)])
def test_device_fresh_init_bit_exact(pr, ctx, S, A, hid, seed):
    a = pr.Agent(ctx, S, A, hid).init_device(seed, lr=3e-4)
    want = pr.artifact_init(S, A, seed, hid).astype(np.float32).astype(np.float64)
    p, m, v, t = a.get()
    assert np.array_equal(p, want)
    assert not np.any(m) and not np.any(v) and t == 0


def test_agent_checkpoint_roundtrip(pr, ctx, tmp_path):
    a = pr.Agent.init(ctx, 181, 30, seed=3)
    a.mutate(5, 0.1)
    rng = np.random.default_rng(0)
    m = rng.normal(size=a.param_count) * 1e-3
    v = rng.uniform(0, 1e-4, a.param_count)
    a.set(a.flatten_params(), m, v, t=42, lr=2.5e-4)
    info = pr.CheckpointInfo(parent_pod=11, mutation_seed=2**64 - 3, algo_tag="ppo", meta=(1.5, 2048.0, 0.25))
    blob = pr.checkpoint_encode(a, info)
    b = pr.Agent(ctx, 181, 30)
    got = pr.checkpoint_decode(b, blob)
    assert got == info
    pa, ma, va, ta = a.get()
    pb, mb, vb, tb = b.get()
    assert np.array_equal(pa, pb) and np.array_equal(ma, mb) and np.array_equal(va, vb) and ta == tb == 42
    assert pr.checkpoint_encode(b, info) == blob  # lr and the Adam hyper-parameters travel too
    path = str(tmp_path / "elite.podrckpt")
    pr.save_checkpoint(a, path, info)
    with open(path, "rb") as f:
        assert f.read() == blob
    c = pr.Agent(ctx, 181, 30)
    assert pr.load_checkpoint(c, path) == info
    assert np.array_equal(c.flatten_params(), pa)
    with pytest.raises(pr.DimensionError):
        pr.checkpoint_decode(pr.Agent(ctx, 181, 30, (32, 32)), blob)


def test_reference_checkpoint_loads(pr, ctx):
    g = np.load(GOLDEN_R2)
    S, A, h = (int(x) for x in g["ck_shape"])
    a = pr.Agent(ctx, S, A, (h,))
    info = pr.checkpoint_decode(a, g["ck_bytes_meta"].tobytes())
    assert (info.parent_pod, info.mutation_seed, info.algo_tag) == (7, 2**63 + 12345, "ppo")
    p, m, v, t = a.get()
    f32 = lambda x: x.astype(np.float32).astype(np.float64)
    assert np.array_equal(p, f32(g["ck_flat"])) and np.array_equal(m, f32(g["ck_m"])) and t == 17
