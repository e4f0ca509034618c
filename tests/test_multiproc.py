"""Multi-process (gloo, world_size 2, CPU) checks of the stream-sharded
driver logic in bench.py: ranks own disjoint streams, the only collectives
are the barrier and the max-of-times reduction, and a stream's tracking
output does not depend on which rank (or how many ranks) processed it."""
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


def _track_stream(seed):
    from oracle import ftoracle as O
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(64, 48, 3, 3, seed=seed, det_every=2)
    st = O.StreamState()
    prm = O.FlowParams(warps_per_level=1, iterations_per_warp=3)
    for t in range(3):
        d = None if dets[t] is None else [O.Det(x.class_id, x.label, x.score, x.box) for x in dets[t]]
        O.step(st, frames[t], t, d, prm)
    return np.array([[o.id, *o.box, o.state == "active"] for o in st.tracks], dtype=np.float64)


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench
    w, r, _ = bench.dist_init()
    assert (w, r) == (ws, rank) and dist.get_backend() == "gloo"
    seeds = [bench.stream_seed(rank, s) for s in range(2)]
    out = {s: _track_stream(s) for s in seeds}
    m = bench.allmax(ws, float(rank + 1))
    bench.barrier(ws)
    q.put((rank, seeds, m, out))
    dist.destroy_process_group()


def test_stream_sharding_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    all_seeds = [s for _, seeds, _, _ in res for s in seeds]
    assert len(set(all_seeds)) == len(all_seeds)  # disjoint shards
    assert all(m == float(ws) for _, _, m, _ in res)  # max over ranks
    for _, _, _, out in res:  # rank-independent per-stream output
        for seed, arr in out.items():
            assert np.array_equal(arr, _track_stream(seed))


@pytest.mark.parametrize("ws", [1])
def test_single_rank_helpers(ws):
    import bench
    assert bench.allmax(ws, 3.5) == 3.5
    assert bench.stream_seed(0, 1) != bench.stream_seed(1, 1)
