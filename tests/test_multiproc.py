"""Multi-process (world_size 2) checks of the stream-sharded multi-GPU path
(paper_1910_06017_b200/shard.py): ranks own disjoint blocks
of global stream ids, the only collectives are the timing barrier, the max
of the ranks' times and the final host gather of track records, and a
stream's output does not depend on which rank (or how many ranks) ran it.

The CPU test runs the sharding / gather logic over gloo.  The GPU test runs
the PRODUCT (a Tracker per rank) as two ranks on cuda:0 over gloo -- the
ranks never wait on each other's kernels, so sharing one GPU only
serialises them -- and checks every stream's tracks against a one-rank run
of all streams."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, ws, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=fn, args=(r, ws, port, q, *args)) for r in range(ws)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in range(ws):
            res.append(q.get(timeout=240))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def _env(rank, ws, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank), FT_DIST_BACKEND="gloo")


def _cpu_worker(rank, ws, port, q):
    _env(rank, ws, port)
    import torch.distributed as dist

    from paper_1910_06017_b200 import _lib, shard
    w, r, _ = shard.init()
    assert (w, r) == (ws, rank) and dist.get_backend() == "gloo"
    ids = shard.shard(rank, ws, total=5)
    recs = []
    for g in ids:  # a fake per-stream record table whose content names its stream
        a = np.zeros(g + 1, dtype=_lib.TRACK_DTYPE)
        a["id"] = np.arange(g + 1)
        a["born_at"] = g
        recs.append(a)
    m = shard.allmax(ws, float(rank + 1))
    shard.barrier(ws)
    got = shard.gather_tracks(ws, rank, ids, recs)
    q.put((rank, ids, m, None if got is None else {k: v.tolist() for k, v in got.items()}))
    dist.destroy_process_group()


def test_shard_and_gather_gloo():
    res = _spawn(_cpu_worker, 2)
    ids = [i for _, part, _, _ in res for i in part]
    assert ids == [0, 1, 2, 3, 4]  # disjoint contiguous blocks, lower ranks first
    assert all(m == 2.0 for _, _, m, _ in res)  # max over ranks
    merged = res[0][3]
    assert res[1][3] is None and sorted(merged) == ids
    for g, rows in merged.items():
        assert len(rows) == g + 1 and all(r[9] == g for r in rows)


def test_shard_blocks():
    from paper_1910_06017_b200 import shard
    assert shard.shard(1, 4, per_rank=64) == list(range(64, 128))
    sizes = [len(shard.shard(r, 3, total=64)) for r in range(3)]
    assert sizes == [22, 21, 21]
    assert sorted(sum((shard.shard(r, 8, total=64) for r in range(8)), [])) == list(range(64))
    assert shard.stream_seed(5) == 1005
    with pytest.raises(ValueError):
        shard.shard(0, 4, total=3)
    with pytest.raises(ValueError):
        shard.shard(0, 2, per_rank=2, total=4)
    assert shard.allmax(1, 3.5) == 3.5


# ---------------------------------------------------------------- GPU: product
GW, GH, GOBJ, GT, GSTREAMS = 128, 96, 4, 4, 4


def _run_streams(ids):
    """Track the given global streams in one Tracker on cuda:0."""
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.shard import stream_seed
    from paper_1910_06017_b200.synth import make_sequence
    seqs = [make_sequence(GW, GH, GOBJ, GT, seed=stream_seed(g), det_every=2, scale_change=True)
            for g in ids]
    trk = Tracker(GW, GH, n_streams=len(ids), device=0, max_tracks=32, max_dets=32,
                  flow_params=FlowParams(warps_per_level=2, iterations_per_warp=9))
    out = []
    for t in range(GT):
        recs = trk.step_records(np.stack([s[0][t] for s in seqs]), t, [s[1][t] for s in seqs])
        frame = []
        for r in recs:  # label handles are per Tracker: compare the label strings
            r = r.copy()
            labels = [trk._label_names[k] for k in r["label_ref"]]
            r["label_ref"] = 0
            frame.append((r, labels))
        out.append(frame)
    trk.close()
    return out


def _gpu_worker(rank, ws, port, q):
    _env(rank, ws, port)
    os.environ["LOCAL_RANK"] = "0"  # both ranks share the box's one GPU
    import torch
    import torch.distributed as dist

    from paper_1910_06017_b200 import shard
    shard.init()
    torch.cuda.set_device(0)
    ids = shard.shard(rank, ws, total=GSTREAMS)
    per_frame = _run_streams(ids)
    got = shard.gather_tracks(ws, rank, ids, per_frame[-1])
    q.put((rank, ids, None if got is None else {k: (v[0].tobytes(), v[1]) for k, v in got.items()}))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_match_one_rank():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    res = _spawn(_gpu_worker, 2)
    assert [r[1] for r in res] == [[0, 1], [2, 3]]
    merged = res[0][2]
    one = _run_streams(list(range(GSTREAMS)))[-1]
    assert sorted(merged) == list(range(GSTREAMS))
    for g in range(GSTREAMS):
        assert merged[g] == (one[g][0].tobytes(), one[g][1]), f"stream {g}: 2 ranks != 1 rank"
    assert sum(len(r) for r, _ in one) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("split,total,scaling", [(["--streams", "2"], 4, "weak"),
                                                 (["--total-streams", "3"], 3, "strong")])
def test_bench_two_ranks_one_gpu(split, total, scaling):
    """bench.py's multi-rank path end to end (`--gpus 2` starts the ranks
    itself): both ranks on cuda:0 over gloo (FT_BENCH_ONE_GPU test hook), a
    tiny weak-scaling run and an uneven strong split (2 + 1 streams); rank 0
    prints one line covering both ranks' streams (functional check, not a
    scaling number)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FT_BENCH_ONE_GPU="1", FT_DIST_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--steps", "2", "--warmup", "3", *split, "--no-cpu-baseline"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == scaling
    assert d["config"]["total_streams"] == total and d["gather"]["streams"] == total
    assert d["value"] > 0 and abs(d["value_per_gpu"] - d["value"] / 2) < 1e-3 * d["value"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
