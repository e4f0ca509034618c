"""Frame period of the pipelined Tracker with and without the device
prefetch, B SD streams (GPU box).  python tools/prefetch_probe.py [B ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1910_06017_b200.pipeline import Tracker  # noqa: E402


def main(Bs):
    import torch
    T = 24
    for B in Bs:
        seqs = [bench.gen_stream(g, T) for g in range(B)]
        frames = [np.stack([seqs[s][0][t] for s in range(B)]) for t in range(T)]
        recs = [[seqs[s][1][t] for s in range(B)] for t in range(T)]
        for pf in (False, True, False, True):
            trk = Tracker(720, 576, n_streams=B, max_tracks=256, max_dets=160, prefetch=pf)
            for t in range(4):
                trk.submit(frames[t], t, recs[t])
                trk.wait()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sub = wai = 0.0
            for t in range(4, T):
                a = time.perf_counter()
                trk.submit(frames[t], t, recs[t])
                b = time.perf_counter()
                if t > 4:
                    trk.wait()
                sub += b - a
                wai += time.perf_counter() - b
            trk.wait()
            torch.cuda.synchronize()
            per = 1000 * (time.perf_counter() - t0) / (T - 4)
            ph = trk.phase_ms(-1)
            print(f"B={B} prefetch={pf}: {per:.3f} ms/frame (submit {1000 * sub / (T - 4):.3f}, "
                  f"wait {1000 * wai / (T - 4):.3f}); phases {ph}", flush=True)
            trk.close()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 8])
