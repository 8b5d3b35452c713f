"""SURVEY.md 8f items on the GPU: the file loader (reference binary format,
sharded), the exact-count tuning service, and the verify / bench commands."""

import csv

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_store_from_file_sharded(gpu, tmp_path):
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 30_001, 6, seed=3))
    path = tmp_path / "d.bin"
    gpu.write_dataset(data, path)
    rng = np.random.default_rng(0)
    lo = (rng.random((20, 6)) * 0.5).astype(np.float32)
    hi = lo + np.float32(0.6)
    exp_offs, exp_ids = oracle.ids_batch(data.values, lo, hi)
    world = 3
    parts = []
    for r in range(world):
        with gpu.DeviceStore.from_file(path, shard=(r, world), layouts=1 | 4) as st:
            parts.append(st.ids(lo, hi, "vafile_batch"))
    # rank-ordered concatenation per query == the whole-table result
    for q in range(lo.shape[0]):
        got = np.concatenate([ids[o[q]:o[q + 1]] for o, ids in parts]).astype(np.int64)
        assert np.array_equal(got, exp_ids[exp_offs[q]:exp_offs[q + 1]]), q


def test_collect_selectivity_buckets_exact(gpu):
    from paper_1801_03644_b200.tuning import collect_selectivity_buckets, selectivities
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 50_000, 3, seed=5))
    buckets = [(0.0, 0.01), (0.05, 0.2)]
    out = collect_selectivity_buckets(data, buckets, per_bucket=10, seed=1, batch=512)
    for (blo, bhi), qs in zip(buckets, out):
        assert len(qs) == 10
        for q in qs:
            exact = oracle.brute_ids(data.values, q.lower, q.upper).size / data.n
            assert blo <= exact <= bhi
        assert np.allclose(selectivities(data, qs),
                           [oracle.brute_ids(data.values, q.lower, q.upper).size / data.n for q in qs])


def test_tune_halfwidth_hits_target(gpu):
    from paper_1801_03644_b200.tuning import tune_halfwidth
    v = np.random.default_rng(2).random((200_000, 4), dtype=np.float32)
    with gpu.DeviceStore(v) as st:
        h = tune_halfwidth(st, v[17], np.array([0, 2]), 0.01)
        lo = np.full(4, -np.inf, np.float32)
        hi = np.full(4, np.inf, np.float32)
        lo[[0, 2]] = v[17, [0, 2]] - h
        hi[[0, 2]] = v[17, [0, 2]] + h
        sel = oracle.brute_ids(v, lo, hi).size / v.shape[0]
        assert 0.005 < sel < 0.02


def test_cli_verify_and_bench(gpu, tmp_path, capsys):
    from paper_1801_03644_b200.cli import main
    assert main(["verify", "--n", "20000", "--dims", "4", "--count", "50",
                 "--method", "sequential,horizontal,vertical,vafile"]) == 0
    text = capsys.readouterr().out
    assert "verification passed" in text
    # the ground truth is computed on the CPU (the reference's own scan when
    # baseline/_ref holds it), never by a GPU kernel
    assert "ground truth: reference SequentialScan(SCALAR)" in text or "ground truth: numpy containment" in text
    out = tmp_path / "r.csv"
    assert main(["bench", "--n", "20000", "--dims", "4", "--count", "50", "--method", "vafile,vertical",
                 "--repetitions", "2", "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0][0] == "method" and len(rows) == 3 and float(rows[1][rows[0].index("qps")]) > 0


def _nccl_one_rank(port, q):
    import os
    import numpy as np
    import torch
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        from paper_1801_03644_b200.parallel import ShardedScan
        rng = np.random.default_rng(5)
        values = rng.random((200_003, 6), dtype=np.float32)
        lo = rng.uniform(0, 0.4, (40, 6)).astype(np.float32)
        hi = (lo + 0.6).astype(np.float32)
        scan = ShardedScan(values, 0, values.shape[0], device=0)
        exp_offs, exp_ids = oracle.ids_batch(values, lo, hi)
        ok = np.array_equal(scan.count_batch(lo, hi), np.diff(exp_offs))
        o, i = scan.search_batch(lo, hi)
        ok &= np.array_equal(o, exp_offs) and np.array_equal(i.astype(np.int64), exp_ids)
        o2, i2, buf = scan.search_batch_host(lo, hi)   # kernel writes into registered shared host memory
        ok &= np.array_equal(o2, exp_offs) and np.array_equal(i2.astype(np.int64), exp_ids)
        del i2
        buf.close()
        scan.close()
        dist.destroy_process_group()
        q.put(bool(ok))
    except Exception as e:
        q.put(repr(e))


def test_sharded_scan_device_path_nccl_one_rank(gpu):
    """ShardedScan's device path under NCCL (one rank: the only GPU here):
    ids stay in HBM through the merge, and the direct host write lands every
    slice at its rank-ordered offset in the registered shared buffer."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank, args=(port, q))
    p.start()
    try:
        res = q.get(timeout=300)
    finally:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert res is True, res
