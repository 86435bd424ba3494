"""G-vs-1 bit-exactness of the multi-process slab path at each stage (init,
run, upload + run), ranks sharing GPUs allowed (gloo control plane).
torchrun --nproc-per-node 2 tools/dist_check.py [n_per_rank] [cols]"""
import os
import sys
import zlib

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_17284_b200 import ltl  # noqa: E402
from paper_2406_17284_b200.dist import PartitionedTorus  # noqa: E402

rows_per = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
rule = "R8,C2,M0,S163..223,B74..252,NM"
G = world * rows_per
part = PartitionedTorus(G, cols, rank, world, dev)
part.init_random(0.23, 1)


def check(tag, gens):
    if os.environ.get("SYNC_BEFORE_CHECK"):
        part.torus.synchronize()
        dist.barrier()
    mine = part.torus.download()
    table = [None] * world
    dist.all_gather_object(table, (part.row0, part.rows, zlib.crc32(memoryview(mine))))
    slabs = [None] * world
    if os.environ.get("DIFF"):
        dist.all_gather_object(slabs, mine)
    if rank == 0:
        with ltl.DeviceTorus(rows=G, cols=cols) as t:
            t.init_random(0.23, 1)
            if gens:
                t.run(rule, gens)
            full = t.download()
        ok = [zlib.crc32(memoryview(np.ascontiguousarray(full[r0:r0 + rr]))) == c for r0, rr, c in table]
        print(f"{tag}: gens {gens} ring={part.ring} persist={part.persist} slabs ok {ok}", flush=True)
        if os.environ.get("DIFF"):
            for (r0, rr, _), sl in zip(table, slabs):
                d = np.argwhere(sl != full[r0:r0 + rr])
                if len(d):
                    rows_bad = np.unique(d[:, 0])
                    print(f"  slab at {r0}: {len(d)} cells differ, rows {rows_bad[:8].tolist()}..{rows_bad[-4:].tolist()}, "
                          f"cols {np.unique(d[:, 1])[:8].tolist()}", flush=True)
    dist.barrier()


if not os.environ.get("SKIP_INIT_CHECK"):
    check("init", 0)
if os.environ.get("DOWNLOAD_ONLY"):  # a download before the run, no reference torus
    if os.environ.get("DOWNLOAD_ONLY") in ("all", str(rank)):
        part.torus.download()
    dist.barrier()
    if os.environ.get("REFILL"):
        part._ring_fill()
if os.environ.get("RECHECK_INIT"):
    check("init again (no run)", 0)
GENS = int(os.environ.get("GENS", "3"))
part.run(rule, GENS)
check("run 3", GENS)
h = part.torus.download()
part.upload(h)
check("after re-upload", 3)
part.run(rule, 3)
check("run 3 more", 6)
dist.destroy_process_group()
