"""Host <-> device transfer components of one run_interior-style call at
32768^2 (pinned host grids): upload, 20 generations, download; bit-packed
transfers vs byte copies (LTL_BYTE_TRANSFERS).  python tools/xfer_time.py [n]"""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2406_17284_b200 import ltl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rule = "R5,C2,M1,S34..58,B34..45,NM"
hin = torch.empty((n, n), dtype=torch.uint8).pin_memory().numpy()
hout = torch.empty((n, n), dtype=torch.uint8).pin_memory().numpy()
with ltl.DeviceTorus(n=n) as t:
    t.init_random(0.21, 1)
    t.download(hin)
    for mode in ("bits", "bytes", "bits", "bytes"):
        if mode == "bytes":
            os.environ["LTL_BYTE_TRANSFERS"] = "1"
        else:
            os.environ.pop("LTL_BYTE_TRANSFERS", None)
        t.upload(hin)
        t.download(hout)  # warm
        t0 = time.perf_counter()
        t.upload(hin)
        t1 = time.perf_counter()
        t.run(rule, 20)
        t2 = time.perf_counter()
        t.download(hout)
        t3 = time.perf_counter()
        t4 = time.perf_counter()
        t.run_interior(hin, rule, 20, out=hout)
        t5 = time.perf_counter()
        print(f"{mode:5s} upload {1e3 * (t1 - t0):6.2f} ms  run {1e3 * (t2 - t1):6.2f} ms  "
              f"download {1e3 * (t3 - t2):6.2f} ms  run_interior {1e3 * (t5 - t4):6.2f} ms", flush=True)
