"""Multi-process slab decomposition on CPU (gloo, world size 2 and 3).

Each rank owns a row slab of one torus with 16 halo rows, advances it with
the oracle on the padded slab, and exchanges boundary rows through
paper_2406_17284_b200.dist.exchange_edges -- the same plan the GPU ranks run
over NCCL.  The assembled grid must equal the single-process oracle run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HALO = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _padded_step(orc, padded, rows, cols, rule):
    """One generation of a padded slab (rows + 32) x (cols + 32): the oracle
    runs on the periodic torus of the padded block, and only interior cells whose
    window stays inside the block are kept -- so the halo rows alone determine
    the slab's boundary rows, exactly as on the device."""
    out = orc.step(padded, rule)
    nxt = padded.copy()
    nxt[HALO:HALO + rows, HALO:HALO + cols] = out[HALO:HALO + rows, HALO:HALO + cols]
    return nxt


def _worker(rank, world, port, global_rows, cols, steps, rule, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2406_17284_b200.dist import HaloPlan, exchange_edges, slab_rows
    orc = oracle.Oracle()
    rng = np.random.default_rng(3)
    full = (rng.random((global_rows, cols)) < 0.3).astype(np.uint8)
    row0, rows = slab_rows(global_rows, world, rank)
    pitch = cols + 2 * HALO
    padded = np.zeros((rows + 2 * HALO, pitch), np.uint8)
    padded[HALO:HALO + rows, HALO:HALO + cols] = full[row0:row0 + rows]
    plan = HaloPlan.ring(rank, world)

    def refresh():
        # local column wrap (ltl_halo.cu for a part), then the packed edge
        # exchange (ltl_pack_edges -> send/recv -> ltl_unpack_halo)
        padded[HALO:HALO + rows, :HALO] = padded[HALO:HALO + rows, cols:cols + HALO]
        padded[HALO:HALO + rows, cols + HALO:] = padded[HALO:HALO + rows, HALO:2 * HALO]
        send_top = torch.from_numpy(padded[HALO:2 * HALO, HALO:HALO + cols].copy())
        send_bot = torch.from_numpy(padded[rows:rows + HALO, HALO:HALO + cols].copy())
        recv_top, recv_bot = torch.empty_like(send_top), torch.empty_like(send_bot)
        exchange_edges(send_top, send_bot, recv_top, recv_bot, plan, dist)
        for rows_dst, got in ((slice(0, HALO), recv_top),
                              (slice(rows + HALO, rows + 2 * HALO), recv_bot)):
            g = got.numpy()
            padded[rows_dst, HALO:HALO + cols] = g
            padded[rows_dst, :HALO] = g[:, cols - HALO:]
            padded[rows_dst, cols + HALO:] = g[:, :HALO]

    refresh()
    for _ in range(steps):
        padded = _padded_step(orc, padded, rows, cols, rule)
        refresh()
    result_q.put((rank, row0, padded[HALO:HALO + rows, HALO:HALO + cols].copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,global_rows,cols", [(2, 64, 48), (3, 96, 40)])
def test_slab_exchange_matches_single_process(world, global_rows, cols):
    import oracle
    rule = [5, 2, 1, 34, 58, 34, 45, 0]
    steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, global_rows, cols, steps, rule, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort()
    assembled = np.concatenate([p[2] for p in parts], axis=0)
    rng = np.random.default_rng(3)
    full = (rng.random((global_rows, cols)) < 0.3).astype(np.uint8)
    expect = oracle.Oracle().simulate(full, rule, steps)
    assert np.array_equal(assembled, expect)


def test_slab_rows_partition():
    from paper_2406_17284_b200.dist import HaloPlan, slab_rows
    for total, world in ((100, 3), (64, 8), (16384 * 8, 8), (17, 1)):
        spans = [slab_rows(total, world, r) for r in range(world)]
        assert spans[0][0] == 0
        for (a0, an), (b0, _) in zip(spans, spans[1:]):
            assert a0 + an == b0
        assert sum(n for _, n in spans) == total
    p = HaloPlan.ring(0, 4)
    assert (p.up, p.down) == (3, 1)
