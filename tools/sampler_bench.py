"""Device throughput of the amplitude consumers (csrc/sampler.cu).

    python tools/sampler_bench.py [n_entries]

Inputs already in HBM (torch CUDA tensors), wall time of the synchronous C-ABI
call over 5 repetitions after 2 warm-ups; algorithmic bytes: committed
indices 8 B/entry written; sample 8 (prob) + 8 (index) read + 1 flag written
+ 1 flag read + 8 (index) read by the compaction + 8 per accepted index;
tail mass 8 read + 8 contrib written, bootstrap 4+4 per pick + 8 per gathered
contrib.  Prints one JSON line.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_10749_b200 import sampler as S  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    nq = 42
    req = S.SampleRequest(n_qubits=nq, count=n // 10, seed=3)
    n = req.batch_size
    d_idx = torch.empty(n, dtype=torch.int64, device="cuda")
    t_commit = timed(lambda: S.LIB.gs_committed_indices(0, nq, 3, 0, n, d_idx.data_ptr()))
    p = torch.empty(n, dtype=torch.float64, device="cuda").exponential_() / float(1 << nq)
    out = np.empty(n, dtype=np.int64)
    t_sample = timed(lambda: S.sample_frugal(req, d_idx, p))
    acc = S.sample_frugal(req, d_idx, p).accepted_count
    m = min(n, 10_000_000)
    pm = p[:m].contiguous()
    t_tail = timed(lambda: S.tail_mass(pm, nq, resamples=10, seed=1), reps=3, warm=1)
    del out
    line = {
        "entries": n,
        "committed_indices": {"ms": t_commit * 1e3, "entries_per_s": n / t_commit, "GB_s": 8 * n / t_commit / 1e9},
        "sample_frugal": {"ms": t_sample * 1e3, "entries_per_s": n / t_sample, "accepted": acc,
                          "GB_s": (34 * n + 8 * acc) / t_sample / 1e9, "note": "includes the accepted-index D2H"},
        "tail_mass": {"entries": m, "resamples": 10, "ms": t_tail * 1e3,
                      "GB_s": (16 * m + 16 * 10 * m) / t_tail / 1e9},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
