"""Throughput of CATSNAP v1 snapshot I/O: the device-
streamed ltl_snapshot_write / ltl_snapshot_read against the reference's
snapshot_write / snapshot_read (oracle/_ref) on the same grid and file system.

    python tools/snapshot_bench.py [--n 16384] [--dir /dev/shm] > profiles/snapshot_r01.json

Payload GB/s = n^2 bytes / wall time of the call (file opened, written /
read, closed; page cache as the OS leaves it -- the same for both sides).
The reference side needs the grid in host memory first (its Grid); that
download is NOT charged to it.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=3):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[16384, 32768])
    ap.add_argument("--dir", default="/dev/shm")
    ap.add_argument("--no-reference", action="store_true")
    args = ap.parse_args()
    import numpy as np
    from paper_2406_17284_b200 import ltl
    ref = None
    if not args.no_reference:
        import oracle
        ref = oracle.Reference()
    for n in args.n:
        path = os.path.join(args.dir, f"ltl_snap_{n}.bin")
        rpath = os.path.join(args.dir, f"ref_snap_{n}.bin")
        with ltl.DeviceTorus(n=n) as t:
            t.init_random(0.21, 1)
            w = timed(lambda: t.snapshot_write(path))
            r = timed(lambda: t.snapshot_read(path))
            grid = t.download()
        line = {"what": "CATSNAP v1 snapshot I/O", "n": n, "bytes": n * n, "dir": args.dir,
                "device_write_s": w, "device_write_gbs": n * n / w / 1e9,
                "device_read_s": r, "device_read_gbs": n * n / r / 1e9}
        if ref is not None:
            rw = timed(lambda: ref.snapshot_write(grid, rpath), reps=1)
            same = os.path.getsize(rpath) == os.path.getsize(path)
            if same:
                with open(path, "rb") as a, open(rpath, "rb") as b:
                    while same:
                        x, y = a.read(1 << 24), b.read(1 << 24)
                        same = x == y
                        if not x:
                            break
            rr = timed(lambda: ref.snapshot_read(rpath), reps=1)
            line.update({"reference_write_s": rw, "reference_write_gbs": n * n / rw / 1e9,
                         "reference_read_s": rr, "reference_read_gbs": n * n / rr / 1e9,
                         "identical_files": bool(same),
                         "reference": "catsim::snapshot_write/read (oracle/_ref), 1 thread"})
            os.unlink(rpath)
        os.unlink(path)
        del grid
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
