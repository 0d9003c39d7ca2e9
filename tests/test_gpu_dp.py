"""The data-parallel Trainer path (optimize.Trainer with world > 1) on the
GPU: two ranks share cuda:0 over gloo (one B200 per gpurun call), each
replays its captured graph on its contiguous shard of the global batch,
all-reduces the flat gradient and applies Adam (optimize.py:299-351
re-hosted).

Checks, deterministic backward:
* the all-reduced gradient equals, bit for bit, the sum of the two
  half-batch gradients that a single-rank Trainer computes (fp32 a + b is
  commutative, so the collective adds nothing beyond that one rounding);
* after several steps both ranks hold bit-identical parameters and Adam
  moments (the replicas never diverge);
* those parameters match a single-rank Trainer on the same global batches
  to fp32 rounding of the batch sum (1e-5).
Also `bench.py --gpus 2` self-launches two ranks and reports n_gpus 2."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W, H, B, STEPS = 90, 30, 8, 3


def _setup():
    oc = O.round_f32(O.perturbed_scene(400, seed=21))
    txs = O.sample_tx(5, 64)
    gts = (np.random.default_rng(4).random((64, H, W, 1)) * 0.3).astype(
        np.float32)
    rng = np.random.default_rng(9)
    batches = [rng.integers(64, size=B) for _ in range(STEPS)]
    return oc, txs, gts, batches


def _trainer(oc, txs, gts, graph=True, batch=B):
    from paper_2511_22793_b200 import GaussianCloud, ViewPose
    from paper_2511_22793_b200.optimize import TrainConfig, Trainer
    cloud = GaussianCloud(*(getattr(oc, k).copy() for k in O.GROUPS))
    cfg = TrainConfig(width=W, height=H, batch_tx=batch, deterministic=True)
    tr = Trainer(cloud, ViewPose(np.zeros(3)), cfg, txs, gts)
    if graph:
        tr.capture()
    return tr


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oc, txs, gts, batches = _setup()
    tr = _trainer(oc, txs, gts)
    assert (tr.rank, tr.world, tr.Bl) == (rank, world, B // world)
    grads = []
    for b in batches:
        tr.step(b)
        torch.cuda.synchronize()
        assert tr.check()
        grads.append(tr.grad.cpu().numpy().copy())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             grads=np.stack(grads), params=_params(tr),
             m=tr.state.m.cpu().numpy(), v=tr.state.v.cpu().numpy())
    dist.destroy_process_group()


def _params(tr):
    return np.concatenate([getattr(tr.dev, k).double().cpu().numpy().ravel()
                           for k in O.GROUPS])


def test_dp_two_ranks_on_one_gpu(tmp_path):
    import torch
    import torch.multiprocessing as mp
    port = 29700 + os.getpid() % 500
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    for k in ("grads", "params", "m", "v"):
        assert np.array_equal(r0[k], r1[k]), f"ranks diverged in {k}"

    # single-rank references on the same global batches
    oc, txs, gts, batches = _setup()
    half = _trainer(oc, txs, gts, graph=False, batch=B // 2)  # no update
    full = _trainer(oc, txs, gts)
    for s, b in enumerate(batches):
        # the DP gradient of step s = g(first half) + g(second half), both
        # evaluated at the parameters the DP run had at step s, which equal
        # `full`'s parameters only to rounding -- so compare step 0 exactly
        # and later steps to tolerance
        if s == 0:
            parts = []
            for sl in (b[:B // 2], b[B // 2:]):
                half.set_batch(sl)
                half._gather()
                half._compute()                 # gradient only, no Adam
                torch.cuda.synchronize()
                parts.append(half.grad.cpu().numpy().copy())
            want = (torch.as_tensor(parts[0]) + torch.as_tensor(parts[1])).numpy()
            assert np.array_equal(r0["grads"][0], want), \
                np.abs(r0["grads"][0] - want).max()
        full.step(b)
    torch.cuda.synchronize()
    assert full.check()
    err = np.abs(r0["params"] - _params(full)).max()
    assert err <= 1e-5, err


@pytest.mark.parametrize("config", ["c1", "c4"])
def test_bench_self_launches_ranks(config):
    """`bench.py --gpus 2` without torchrun launches two ranks (here they
    share the one visible GPU over gloo; the line records that)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", config, "--steps", "6",
                        "--warmup", "3", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines()
                       if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2, line
    assert line["value"] > 0
    if config == "c4":
        assert line["healthy"], line
        assert line["config"]["per_rank_batch"] == 16
