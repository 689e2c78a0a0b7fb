"""Multi-rank path partitioning + reduce, world size 2 on CPU (gloo).

The product path (paper_1807_10749_b200/distributed.py) shards the sorted
retained prefixes into contiguous per-rank ranges and all-reduces the
complex128 partials (NCCL on the GPU box).  Here each rank computes its
partial with the CPU oracle and the reduce runs over gloo; the sum must equal
the single-process result (reference semantics: orchestrator.py:80-85 shard,
:340-342 merge).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_10749_b200 import configs
from paper_1807_10749_b200.distributed import partition_prefixes, sharded_sum


def test_partition_is_contiguous_cover():
    pre = np.random.default_rng(0).choice(10_000, size=777, replace=False)
    for world in (1, 2, 3, 8):
        parts = [partition_prefixes(pre, world, r) for r in range(world)]
        np.testing.assert_array_equal(np.concatenate(parts), np.sort(pre))
        sizes = [p.size for p in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition_prefixes(pre, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pathsum_oracle as oracle

    circ, plan, req, pre = configs.build(name)

    def partial(mine):
        amps = oracle.run_batched(circ, plan, req, mine) if mine.size else np.zeros(req.size, complex)
        return torch.from_numpy(np.ascontiguousarray(amps).view(np.float64).copy())

    total = sharded_sum(partial, pre)
    if rank == 0:
        np.save(out_path, total.numpy().view(np.complex128))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1", "cfg1v2"])
def test_world2_gloo_sum_matches_single_process(tmp_path, name):
    from oracle import pathsum_oracle as oracle

    out = str(tmp_path / "total.npy")
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    got = np.load(out)
    circ, plan, req, pre = configs.build(name)
    want = oracle.run_batched(circ, plan, req, pre)
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-14)


def _repro_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1807_10749_b200.distributed import reproducible_sum

    total = reproducible_sum(_order_sensitive_partial, np.arange(1000))
    if rank == 0:
        np.save(out_path, total.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _order_sensitive_partial(mine):
    # magnitudes spread over 16 decades: any change of summation order shows in the bits
    v = np.zeros(64)
    for p in mine:
        rng = np.random.default_rng(int(p))
        v += rng.standard_normal(64) * 10.0 ** rng.integers(-8, 8, size=64)
    return torch.from_numpy(v)


@pytest.mark.parametrize("world", [2, 4])
def test_reproducible_sum_is_bitwise_equal_across_world_sizes(tmp_path, world):
    from paper_1807_10749_b200.distributed import reproducible_sum

    single = reproducible_sum(_order_sensitive_partial, np.arange(1000)).numpy()
    out = str(tmp_path / "total.npy")
    mp.spawn(_repro_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    assert np.array_equal(got.view(np.uint64), single.view(np.uint64))
    plain = _order_sensitive_partial(np.arange(1000)).numpy()
    np.testing.assert_allclose(got, plain, rtol=1e-9, atol=1e-6)



@pytest.mark.gpu
def test_reproducible_sharded_run_on_device():
    """One rank evaluates all 8 fixed slices on the GPU; the slice-order sum is
    deterministic and matches the plain engine run."""
    from paper_1807_10749_b200.distributed import run_batched_sharded
    from paper_1807_10749_b200.pathsum import run_approx

    circ, plan, req, pre = configs.build("cfg1")
    a = run_batched_sharded(circ, plan, req, device=0, reproducible=True)
    b = run_batched_sharded(circ, plan, req, device=0, reproducible=True)
    assert np.array_equal(a.amps.view(np.uint64), b.amps.view(np.uint64))
    want = run_approx(circ, plan, req, device=0).amps
    np.testing.assert_allclose(a.amps, want, rtol=1e-9, atol=1e-12)


def _device_worker(rank, world, port, name, window, out_dir):
    """One rank of the product path: run_batched_sharded on cuda:0 over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1807_10749_b200.distributed import run_batched_sharded

    circ, plan, req, _ = configs.build(name)
    pre = plan.retained[:window]
    plain = run_batched_sharded(circ, plan, req, prefixes=pre, device=0, dst=None)
    repro = run_batched_sharded(circ, plan, req, prefixes=pre, device=0, dst=None, reproducible=True)
    np.save(os.path.join(out_dir, f"plain{rank}.npy"), plain.amps)
    np.save(os.path.join(out_dir, f"repro{rank}.npy"), repro.amps)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name,window", [("cfg3", 64), ("cfg1", None)])
def test_world2_product_path_on_device(tmp_path, name, window):
    """run_batched_sharded itself with two ranks (two processes sharing cuda:0;
    the reduce runs over gloo on the CUDA partials -- the box has one GPU, so
    NCCL's one-rank-per-GPU rule leaves gloo as the two-rank transport).  Plain
    mode equals the one-process engine run; the reproducible mode is bitwise
    equal to its world-1 result (orchestrator.py:340-342 fold semantics)."""
    from paper_1807_10749_b200.distributed import run_batched_sharded
    from paper_1807_10749_b200.pathsum import run_batched

    circ, plan, req, _ = configs.build(name)
    pre = plan.retained if window is None else plan.retained[:window]
    out = str(tmp_path)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_device_worker, args=(r, 2, port, name, window or len(pre), out))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    single = run_batched(circ, plan, req, prefixes=pre).amps
    world1 = run_batched_sharded(circ, plan, req, prefixes=pre, device=0, reproducible=True).amps
    for r in range(2):
        plain = np.load(os.path.join(out, f"plain{r}.npy"))
        repro = np.load(os.path.join(out, f"repro{r}.npy"))
        assert np.linalg.norm(single) > 0
        assert np.linalg.norm(plain - single) <= 1e-12 * np.linalg.norm(single)
        assert np.array_equal(repro.view(np.uint64), world1.view(np.uint64))
