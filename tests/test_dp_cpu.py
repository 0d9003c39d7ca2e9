"""Multi-process data-parallel plumbing on CPU (gloo, world_size 2): the
sharded, all-reduced gradient equals the single-process sum over the global
batch, and the Adam update that follows is identical on every rank.  The
per-TX gradients come from the CPU oracle (test infrastructure); the code
under test is paper_2511_22793_b200.dp (sharding + flat all-reduce)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

W, H = 36, 9


def _scene():
    oc = O.perturbed_scene(12, seed=5)
    txs = O.sample_tx(9, 4)
    U = np.random.default_rng(3).normal(size=(4, H, W, 2))
    return oc, txs, U


def _flat_grad(oc, tx, U):
    _, aux = O.forward(oc, np.zeros(3), np.eye(3), tx, W, H,
                       dtype=np.float64)
    g = O.backward(U, oc, tx, aux)
    return np.concatenate([g[k].reshape(-1) for k in O.GROUPS])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_22793_b200 import dp
    oc, txs, U = _scene()
    r, w = dp.world()
    assert (r, w) == (rank, world)
    mine = dp.shard(np.arange(4), r, w)
    local = sum(_flat_grad(oc, txs[i], U[i]) for i in mine)
    flat = torch.as_tensor(local)
    dp.allreduce_sum(flat)
    out[rank] = flat.numpy()
    dist.destroy_process_group()


def test_sharded_allreduce_equals_global_sum():
    oc, txs, U = _scene()
    want = sum(_flat_grad(oc, txs[i], U[i]) for i in range(4))
    port = 29500 + os.getpid() % 1000
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        assert np.allclose(out[r], want, rtol=1e-12, atol=1e-14)
    assert np.array_equal(out[0], out[1])


def test_shard_contiguous_and_divisibility():
    from paper_2511_22793_b200 import dp
    gi = np.arange(32)
    parts = [dp.shard(gi, r, 4) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), gi)
    with pytest.raises(ValueError):
        dp.shard(np.arange(6), 0, 4)


def test_sample_stream_matches_reference_order():
    """optimize.sample_stream reproduces optimize.py:327-334 draws."""
    from paper_2511_22793_b200.optimize import TrainConfig, sample_stream
    cfg = TrainConfig(seed=3)
    rng = np.random.Generator(np.random.PCG64(3))
    want = [int(rng.integers(10)) for _ in range(7)]
    got = [b[0] for b in sample_stream(10, cfg, 0, 7, 1)]
    assert got == want
    cfg = TrainConfig(seed=4, deterministic=True)
    rng = np.random.Generator(np.random.PCG64(4))
    order, want = None, []
    for step in range(12):
        pos = step % 5
        if pos == 0 or order is None:
            order = rng.permutation(5)
        want.append(int(order[pos]))
    got = [b[0] for b in sample_stream(5, cfg, 0, 12, 1)]
    assert got == want


def test_gspc_roundtrip_matches_reference_format(tmp_path):
    from paper_2511_22793_b200 import load_checkpoint, save_checkpoint
    from conftest import golden, golden_cloud
    fx = golden("generators")
    ref = golden_cloud(fx, "bench_")
    from paper_2511_22793_b200 import GaussianCloud
    c = GaussianCloud(*(getattr(ref, k) for k in O.GROUPS), mlp_dims=ref.mlp_dims)
    p = tmp_path / "a.gspc"
    save_checkpoint(p, c)
    p2 = tmp_path / "b.gspc"
    O.write_gspc(p2, ref)
    assert p.read_bytes() == p2.read_bytes()
    back = load_checkpoint(p)
    for k in O.GROUPS:
        assert np.array_equal(getattr(back, k), getattr(ref, k))
    with pytest.raises(ValueError, match="bad magic"):
        (tmp_path / "c.gspc").write_bytes(b"XXXX" + p.read_bytes()[4:])
        load_checkpoint(tmp_path / "c.gspc")
    with pytest.raises(ValueError, match="truncated"):
        (tmp_path / "d.gspc").write_bytes(p.read_bytes()[:-8])
        load_checkpoint(tmp_path / "d.gspc")
