"""Host-side logic of bench.py: pair sharding (static rid % pairs rule)
and the max-over-ranks timing reduction, exercised with a world-size-2 gloo group."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

sys.path.insert(0, ROOT)


def test_pair_sharding_partitions_the_trace():
    import bench
    from paper_2509_17357_b200 import engine as E
    t = E.synth_trace(40, 1014, 247, E.ALL_AT_ZERO, 0, 1)
    for pairs in (1, 2, 4):
        parts = [bench.pair_trace(t, p, pairs) for p in range(pairs)]
        ids = np.sort(np.concatenate([x.ids for x in parts]))
        assert np.array_equal(ids, np.sort(t.ids))
        for p, x in enumerate(parts):
            assert (x.ids % pairs == p).all()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = torch.tensor([10.0 + rank * 5.0, 20.0 - rank])  # per-step ms on this rank
    dist.all_reduce(local, op=dist.ReduceOp.MAX)
    done = torch.tensor([100.0 if rank % 2 == 0 else 0.0])  # only pair drivers count requests
    dist.all_reduce(done)
    if rank == 0:
        out.put((local.tolist(), done.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    times, done = q.get(timeout=5)
    assert times == [15.0, 20.0] and done == 100.0


def test_kernel_classes_and_roofline_math():
    """bench.py's CUPTI kernel classing and the roofline object (HBM and tensor classes,
    partition-normalised tensor fraction, traffic scaled from the committed ncu ratios)."""
    import bench
    assert bench.kernel_class("void <unnamed>::gemm_tc_kernel<16>(CUtensorMap_st, ...)") == "gemm_stream"
    assert bench.kernel_class("void <unnamed>::gemm_tc_kernel<256>(CUtensorMap_st, ...)") == "gemm_tc"
    assert bench.kernel_class("void <unnamed>::gemm_tc_kernel<256, 2>(CUtensorMap_st, ...)") == "gemm_tc"
    assert bench.kernel_class("void <unnamed>::gemm_tc_kernel<16, 1>(CUtensorMap_st, ...)") == "gemm_stream"
    assert bench.kernel_class("void <unnamed>::attn_decode_tma_kernel<4, 3>(...)") == "decode_attn"
    assert bench.kernel_class("<unnamed>::attn_prefill_pp_kernel(...)") == "prefill_attn"
    assert bench.kernel_class("<unnamed>::rmsnorm_kernel(...)") == "other"
    stats = {
        "cpi": {"gemm_stream": {"launches": 10, "ms": 0.1, "bytes": 5e8, "flops": 0.0},
                "other": {"launches": 5, "ms": 1.0, "bytes": 0.0, "flops": 0.0}},
        "ppi": {"gemm_tc": {"launches": 2, "ms": 1.0, "flops": 6e14, "bytes": 0.0},
                "prefill_attn": {"launches": 1, "ms": 0.0, "flops": 1e9, "bytes": 0.0}},
    }
    part = {"device_sms": 148, "ppi_sms": 40, "cpi_sms": 108}
    top, classes = bench.roofline(stats, part)
    names = [c["kernel"] for c in classes]
    assert names == ["ppi.gemm_tc", "cpi.gemm_stream"]  # by share; zero-time and 'other' skipped
    hbm = next(c for c in classes if c["kernel"] == "cpi.gemm_stream")
    assert abs(hbm["achieved"] - 5e8 / 10 / 1e-5 / 1e9) < 1e-6 * hbm["achieved"]  # GB/s per launch
    ten = classes[0]
    assert ten["bound"] == "tensor" and abs(ten["frac_partition"] - ten["frac"] * 148 / 40) < 1e-3
    assert top["kernel"] == "ppi.gemm_tc" and "peak_source" in top


def test_pooled_p99_across_pairs():
    """Nearest-rank P99 over TTFT values and TBT samples pooled across every pair's records
    (metrics.cpp:13-20, 35-57), not rank 0's pair alone."""
    import bench
    a = {"records": [{"ttft_ms": 10.0, "tbt_samples_ms": [1.0, 2.0]}, {"ttft_ms": 30.0, "tbt_samples_ms": [3.0]}]}
    b = {"records": [{"ttft_ms": 20.0, "tbt_samples_ms": [50.0] * 3}, {"ttft_ms": -1.0, "tbt_samples_ms": [99.0]}]}
    got = bench.pooled([a, b])
    assert got["requests"] == 3 and got["tbt_samples"] == 6
    assert got["ttft_p99_ms"] == 30.0 and got["tbt_p99_ms"] == 50.0
    assert bench.pooled([a])["tbt_p99_ms"] == 3.0  # one pair alone would miss pair b's tail
    assert bench.nearest_rank(list(range(1, 101))) == 99 and bench.nearest_rank([]) is None


def test_pass_roofline_and_critical_worker():
    import bench
    st = {"pass_weight_bytes": 15e9, "kv_bytes_per_token": 131072,
          "iteration_shapes": {"decode 1-16": [10, 30.0, 4.0, 1000.0], "chunk+1-16": [3, 30.0, 5.0, 100.0]}}
    out = bench.pass_rooflines(st)
    assert list(out) == ["1-16 decoders"]
    d = out["1-16 decoders"]
    assert abs(d["achieved_GBps"] - (15e9 + 4 * 1000 * 131072) / 3000.0 / 1e3) < 0.1
    stats = {"cpi": {"decode_attn": {"launches": 2, "ms": 1.0, "bytes": 1e9, "flops": 0.0}},
             "ppi": {"gemm_tc": {"launches": 2, "ms": 5.0, "flops": 6e14, "bytes": 0.0}}}
    top, classes = bench.roofline(stats, None, critical="cpi")
    assert top["kernel"] == "cpi.decode_attn" and classes[0]["kernel"] == "ppi.gemm_tc"
