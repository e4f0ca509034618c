"""B200-native OmniTrack tracking hot path (arXiv 1910.06017).

Drop-in for the reference `flowtrack` per-frame path: the public modules
mirror flowtrack.{imaging,optflow,track,assoc,detect} and add
pipeline.Tracker (frame in, tracks out).  Compute runs in hand-written
sm_100a CUDA kernels behind the C ABI declared in include/omnitrack.h
(libomnitrack.so), reached through ctypes; torch is used only for device
memory and streams.
"""

__version__ = "0.1.0"
