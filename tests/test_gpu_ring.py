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


def _worker(rank, world, port, global_rows, cols, steps, text, q, multi=False, own_gpu=False,
            race=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if multi:  # multi-generation launches even on small slabs (world 1: self-ring)
        os.environ["LTL_FORCE_PERSIST"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = rank if own_gpu else 0
        torch.cuda.set_device(dev)
        from paper_2406_17284_b200.dist import PartitionedTorus
        part = PartitionedTorus(global_rows, cols, rank, world, dev, ring=True)
        assert part.ring and part.torus.ring_active()
        rng = np.random.default_rng(7)
        full = (rng.random((global_rows, cols)) < 0.3).astype(np.uint8)
        part.upload(np.ascontiguousarray(full[part.row0:part.row0 + part.rows]))
        if race:
            # downloads with no barrier around them, right before and right
            # after the steps: a neighbour may still be reading this rank's
            # buffers (ltl_download must wait for it, never race it)
            part.torus.download()
            part.run(text, 2)
            part.torus.download()
            part.run(text, steps - 2)
        elif multi:
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


@pytest.mark.parametrize("world,global_rows,cols,multi,own_gpu,race", [
    (2, 256, 256, False, False, False), (4, 512, 128, False, False, False),
    (1, 96, 384, False, False, False),
    (2, 256, 256, True, False, False),        # same GPU: one launch per generation
    (1, 512, 384, True, False, False),        # self-ring: persistent ring kernel
    # unsynchronised downloads between steps, multi-band slabs
    (2, 2048, 1024, False, False, True), (4, 2048, 512, False, False, True),
    # one process per GPU (needs >= 2 / 4 GPUs): the cross-device persistent
    # ring kernel, rows pulled over NVLink through CUDA IPC
    (2, 1024, 512, True, True, False), (2, 512, 256, False, True, False),
    (4, 2048, 256, True, True, False), (2, 4096, 1024, True, True, True),
])
def test_ring_processes_match_oracle(orc, world, global_rows, cols, multi, own_gpu, race):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if own_gpu and torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    text = "R16,C2,M0,S170..296,B170..300,NM"
    steps = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, global_rows, cols, steps, text, q, multi, own_gpu,
                               race))
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


@pytest.mark.parametrize("gpus", [2, 4, 8])
def test_slabs_on_several_devices_in_one_process(orc, gpus):
    """One process driving G GPUs (ltl_create with dev_ids 0..G-1): peer access,
    per-device kernel attributes, the in-process ring -- equal to one slab."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    from paper_2406_17284_b200 import ltl
    n, text = 2048, "R8,C2,M0,S163..223,B74..252,NM"
    with ltl.DeviceTorus(n=n) as t:
        t.init_random(0.23, 1)
        init = t.download()
        t.run(text, 6)
        want = t.download()
    with ltl.DeviceTorus(n=n, slabs=gpus, devices=list(range(gpus))) as t:
        t.upload(init)
        t.run(text, 6)
        assert np.array_equal(t.download(), want)
