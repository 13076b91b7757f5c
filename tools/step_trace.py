#!/usr/bin/env python
"""Diagnostics: per-call wall times of the bench step (words workload) to
locate host-side stalls.  Prints one line per step: device ms (events) and
wall ms of the range call, the kNN call and the frees."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import argparse
    args = argparse.Namespace(n=0, nq=0, workload="words")
    w = bench.make_workload("words", 0, args)
    eng = bench.Engine(w, 0)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    eng.upload(sp)
    for i in range(24):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        hs = eng.step_device(sp)
        t1 = time.perf_counter()
        eng.free(hs)
        t2 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"step {i:2d} device {e0.elapsed_time(e1):8.2f} ms  calls {1e3*(t1-t0):8.2f}  free {1e3*(t2-t1):6.2f}  "
              f"sync {1e3*(t3-t2):6.2f}", flush=True)


if __name__ == "__main__":
    main()
