"""Multi-process plumbing of the motion-index data parallelism on CPU:
torch.distributed with the gloo backend, world_size 2 (and 3), fake per-motion
results in place of the kernels.  Checks that contiguous sharding covers every
motion exactly once, that the in-place all-gather assembles the same arrays a
single process would produce (including padded tails), and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_23960_b200 import dist as D


def fake_valid(m):
    return ((m * 2654435761) >> 7) % 3 == 0


def fake_key(m):
    return np.where(m % 5 == 0, 0xFFFFFFFF, (m * 40503) % 66000).astype(np.uint32)


@pytest.mark.parametrize("M", [0, 1, 7, 64, 1000, 1 << 20])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_covers_every_motion_once(M, world):
    seen = np.zeros(M, np.int32)
    pers = set()
    for r in range(world):
        lo, hi, per = D.shard(M, r, world)
        assert 0 <= lo <= hi <= M and hi - lo <= per
        seen[lo:hi] += 1
        pers.add(per)
    assert (seen == 1).all() and len(pers) == 1


def test_pad_rows():
    x = torch.arange(12, dtype=torch.float32).reshape(3, 4)
    y = D.pad_rows(x, 5)
    assert y.shape == (5, 4) and torch.equal(y[:3], x) and torch.equal(y[3], x[0])
    assert D.pad_rows(x, 3) is x


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, M, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"] = str(rank)
    os.environ["WORLD_SIZE"] = str(world)
    os.environ["LOCAL_RANK"] = str(rank)
    r, w, _ = D.init_from_env("gloo")
    assert (r, w) == (rank, world)
    lo, hi, per = D.shard(M, rank, world)
    valid_all = torch.zeros(world * per, dtype=torch.uint8)
    key_all = torch.zeros(world * per, dtype=torch.int32)
    # "kernel": write this rank's results straight into its slice (padding gets garbage)
    m = np.arange(lo, lo + per)
    valid_all[rank * per:(rank + 1) * per] = torch.from_numpy(fake_valid(m).astype(np.uint8))
    key_all[rank * per:(rank + 1) * per] = torch.from_numpy(fake_key(m).view(np.int32))
    D.gather_inplace(valid_all, per, rank, world)
    D.gather_inplace(key_all, per, rank, world)
    t = D.max_over_ranks(float(rank + 1) * 1.5, world)
    per_rank = D.all_ranks(float(rank + 1) * 1.5, world)
    np.save(os.path.join(out_dir, f"p{rank}.npy"), np.array(per_rank))
    np.save(os.path.join(out_dir, f"v{rank}.npy"), valid_all[:M].numpy())
    np.save(os.path.join(out_dir, f"k{rank}.npy"), key_all[:M].numpy().view(np.uint32))
    np.save(os.path.join(out_dir, f"t{rank}.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 1000), (2, 4096), (3, 1001)])
def test_gloo_inplace_allgather_matches_single_process(tmp_path, world, M):
    mp.spawn(_worker, args=(world, M, _free_port(), str(tmp_path)), nprocs=world, join=True)
    m = np.arange(M)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"v{r}.npy"), fake_valid(m).astype(np.uint8))
        assert np.array_equal(np.load(tmp_path / f"k{r}.npy"), fake_key(m))
        assert np.load(tmp_path / f"t{r}.npy")[0] == 1.5 * world      # max over ranks
        assert np.array_equal(np.load(tmp_path / f"p{r}.npy"), 1.5 * np.arange(1, world + 1))   # every rank's


def test_bench_reference_arm_exits_on_nonzero_rank(monkeypatch, capsys):
    import importlib
    import sys
    sys.argv = ["bench.py", "--impl", "reference"]
    monkeypatch.setenv("RANK", "1")
    bench = importlib.import_module("bench")
    bench.run_reference(bench.args_())
    assert capsys.readouterr().out == ""


def test_bench_reference_arm_prints_one_json_line(monkeypatch, capsys):
    import importlib
    import json
    import sys
    sys.argv = ["bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1",
                "--ref-seconds", "0.05"]
    monkeypatch.setenv("RANK", "0")
    bench = importlib.import_module("bench")
    bench.run_reference(bench.args_())
    out = capsys.readouterr().out.strip().splitlines()
    assert len(out) == 1
    d = json.loads(out[0])
    assert d["impl"] == "reference" and d["unit"] == "robot-states/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_time_windows_partition_horizon():
    for T in (1, 31, 32, 1000, 100003):
        for world in (1, 2, 3, 8):
            covered = np.zeros(T, np.int32)
            for r in range(world):
                t0, t1 = D.time_window(T, r, world)
                assert (t0 % 32 == 0 or t0 == T) and t0 <= t1
                covered[t0:t1] += 1
            assert (covered == 1).all()


def _worker_min(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    D.init_from_env("gloo")
    NONE = -1   # 0xFFFFFFFF as int32
    per_rank = {0: [NONE, 5, 2 ** 31 + 7 - 2 ** 32, NONE], 1: [3, NONE, 2 ** 31 + 3 - 2 ** 32, NONE]}
    keys = torch.tensor(per_rank[rank], dtype=torch.int32)
    got = D.allreduce_min_keys(keys, world)
    valid = torch.tensor([1, 0, 1, 1], dtype=torch.uint8) if rank == 0 else torch.tensor([1, 1, 0, 1], dtype=torch.uint8)
    v = D.allreduce_and_valid(valid, world)
    np.save(os.path.join(out_dir, f"m{rank}.npy"), got.numpy().view(np.uint32))
    np.save(os.path.join(out_dir, f"v{rank}.npy"), v.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_min_of_uint32_keys_and_valid(tmp_path):
    mp.spawn(_worker_min, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert np.load(tmp_path / f"m{r}.npy").tolist() == [3, 5, 2 ** 31 + 3, 0xFFFFFFFF]
        assert np.load(tmp_path / f"v{r}.npy").tolist() == [1, 0, 0, 1]
