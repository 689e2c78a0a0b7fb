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
