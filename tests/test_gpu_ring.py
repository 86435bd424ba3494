"""The fused ring halo exchange across PROCESSES (one process per GPU in a real
run), exercised on one B200: 2 and 4 processes share cuda:0, exchange their
CUDA IPC handles over gloo and step with the halo rows pulled by the kernels
out of each other's buffers; at world size 1 the slab is its own neighbour
(and may take the multi-generation ring kernel).  The assembled torus must
equal the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_data import parse_rule_text

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, global_rows, cols, steps, text, q, multi=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if multi:  # multi-generation launches even on small slabs (world 1: self-ring)
        os.environ["LTL_FORCE_PERSIST"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2406_17284_b200.dist import PartitionedTorus
        part = PartitionedTorus(global_rows, cols, rank, world, 0, ring=True)
        assert part.ring and part.torus.ring_active()
        rng = np.random.default_rng(7)
        full = (rng.random((global_rows, cols)) < 0.3).astype(np.uint8)
        part.upload(np.ascontiguousarray(full[part.row0:part.row0 + part.rows]))
        if multi:
            part.run(text, steps - 2)  # all generations in one call ...
            part.run(text, 2)          # ... and a second call continuing the counters
        else:
            for _ in range(steps):
                part.step(text)
        part.torus.synchronize()
        q.put((rank, part.row0, part.torus.download()))
        dist.barrier()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, -1, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,global_rows,cols,multi", [
    (2, 256, 256, False), (4, 512, 128, False), (1, 96, 384, False),
    (2, 256, 256, True),                      # same GPU: one launch per generation
    (1, 512, 384, True),                      # self-ring: persistent ring kernel
])
def test_ring_processes_match_oracle(orc, world, global_rows, cols, multi):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    text = "R16,C2,M0,S170..296,B170..300,NM"
    steps = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, global_rows, cols, steps, text, q, multi))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, row0, out in got:
        assert row0 >= 0, f"rank {rank}: {out}"
    assembled = np.zeros((global_rows, cols), np.uint8)
    for _, row0, out in got:
        assembled[row0:row0 + out.shape[0]] = out
    rng = np.random.default_rng(7)
    full = (rng.random((global_rows, cols)) < 0.3).astype(np.uint8)
    assert np.array_equal(assembled, orc.simulate(full, parse_rule_text(text), steps))
