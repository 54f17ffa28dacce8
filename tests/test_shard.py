"""Multi-process (gloo, world_size 2, CPU) tests of the config-4 sharding and
result gather used by bench.py's batched workload on NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0901_1696_b200.shard import gather_results, shard_range


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e = shard_range(total, rank, world)
    idx = torch.arange(s, e)
    info = (idx % 5 == 3).to(torch.int32) * (idx % 64 + 1).to(torch.int32)
    resid = idx.to(torch.float64) * 1e-3
    gi, gr = gather_results(info, resid, total)
    if rank == 0:
        q.put((gi.tolist(), gr.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 11, 1])
def test_gather_results_gloo_world2(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    gi, gr = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    idx = torch.arange(total)
    want_i = ((idx % 5 == 3).to(torch.int32) * (idx % 64 + 1).to(torch.int32)).tolist()
    assert gi == want_i
    assert gr == pytest.approx((idx.to(torch.float64) * 1e-3).tolist())


def _bench_worker(rank, world, port, q):
    """bench.py's own rank plumbing (dist_setup, barrier, max_over_ranks,
    all_ranks) under gloo, driven through the environment torchrun sets."""
    import importlib.util
    import sys
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "BENCH_DIST_BACKEND": "gloo"})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    sys.modules["bench_under_test"] = bench
    spec.loader.exec_module(bench)
    r, w, local = bench.dist_setup()
    assert (r, w, local) == (rank, world, rank)
    bench.barrier(w)
    mx = bench.max_over_ranks(10.0 + rank, w)      # per-rank ms -> the job's time
    allv = bench.all_ranks(1.5 * (rank + 1), w)    # per_rank_ms of the batched block
    bench.barrier(w)
    if rank == 0:
        q.put((mx, allv))
    dist.destroy_process_group()


def test_bench_rank_helpers_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    mx, allv = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert mx == 11.0
    assert allv == [1.5, 3.0]


def test_bench_reference_arm_other_ranks_exit_without_work():
    """`bench.py --impl reference` under torchrun: ranks != 0 print nothing and
    exit 0 without joining a process group (rank 0 alone times the CPU path)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(_free_port()))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""
