"""Row-slab partitioning of one torus across processes (one per GPU).

Rank k of W owns global rows [k*R, (k+1)*R) with all columns.
One generation = the fused step kernel on every rank (ltl_step_part: main
kernel + local column wrap), then the only exchange the stencil needs: the
16 boundary rows of each slab go to the ring neighbours' halos

    my first 16 interior rows   -> rank-1's 16 halo rows below
    my last 16 interior rows    -> rank+1's 16 halo rows above

packed on the device into contiguous 16 x cols buffers (ltl_pack_edges),
sent with NCCL send/recv on the same stream as the kernels -- no host
synchronisation -- and unpacked into the strip layout with their column wrap
(ltl_unpack_halo).  The same plan drives CPU tensors over gloo in the
world-size-2 tests.
"""
from __future__ import annotations

from dataclasses import dataclass

HALO = 16


@dataclass(frozen=True)
class HaloPlan:
    rank: int
    world: int
    up: int     # rank holding the rows just above mine (global row0 - 1)
    down: int   # rank holding the rows just below mine

    @classmethod
    def ring(cls, rank: int, world: int) -> "HaloPlan":
        return cls(rank, world, (rank - 1) % world, (rank + 1) % world)


def slab_rows(global_rows: int, world: int, rank: int):
    """(row0, rows) of rank's slab; remainder rows go to the first ranks."""
    base, extra = divmod(global_rows, world)
    rows = base + (1 if rank < extra else 0)
    row0 = rank * base + min(rank, extra)
    return row0, rows


def exchange_edges(send_top, send_bot, recv_top, recv_bot, plan: HaloPlan, dist_mod=None) -> None:
    """The per-generation exchange of a row-slab partition.

    send_top: my first 16 interior rows   -> the upper neighbour's bottom halo
    send_bot: my last 16 interior rows    -> the lower neighbour's top halo
    recv_top: <- the upper neighbour's last 16 rows  (my 16 halo rows above)
    recv_bot: <- the lower neighbour's first 16 rows (my 16 halo rows below)

    All four are contiguous 16 x cols byte tensors (CUDA for NCCL, CPU for
    gloo); the device packs / unpacks them from its strip layout
    (ltl_pack_edges / ltl_unpack_halo).
    """
    if dist_mod is None:
        import torch.distributed as dist_mod  # noqa: N813
    if plan.world == 1:
        recv_top.copy_(send_bot)
        recv_bot.copy_(send_top)
        return
    ops = [
        dist_mod.P2POp(dist_mod.isend, send_top, plan.up),
        dist_mod.P2POp(dist_mod.irecv, recv_bot, plan.down),
        dist_mod.P2POp(dist_mod.isend, send_bot, plan.down),
        dist_mod.P2POp(dist_mod.irecv, recv_top, plan.up),
    ]
    # With world == 2 both neighbours are the same rank; messages between a
    # pair match in issue order, and every rank issues (top, bottom) sends and
    # (bottom, top) receives, which pairs my top rows with the peer's bottom
    # halo and vice versa.
    for req in dist_mod.batch_isend_irecv(ops):
        req.wait()


class PartitionedTorus:
    """One rank's slab of a torus split across processes, driven through the C-ABI.

    Two exchange paths for the 16 boundary rows per generation:
      * ring (cols % 128 == 0, slab rows % 32 == 0): fused into the step --
        the kernel's first / last band units TMA-load the 16 rows beyond the
        slab straight out of the ring neighbours' slabs (CUDA IPC peer memory
        over NVLink) once the neighbours' step counters say that generation
        is complete.  No NCCL on the data path, no extra launches, no host
        synchronisation;
      * otherwise: ltl_pack_edges -> NCCL send/recv (exchange_edges) ->
        ltl_unpack_halo on the same stream.
    """

    def __init__(self, global_rows: int, cols: int, rank: int, world: int, device: int,
                 ring: bool | None = None, dist_mod=None):
        from .ltl import DeviceTorus
        if dist_mod is None:
            import torch.distributed as dist_mod  # noqa: N813
        self.dist = dist_mod
        self.plan = HaloPlan.ring(rank, world)
        self.row0, self.rows = slab_rows(global_rows, world, rank)
        if world > 1 and self.rows < HALO:
            raise ValueError("geometry error: slab thinner than the 16-row halo")
        self.cols = cols
        self.torus = DeviceTorus(rows=self.rows, cols=cols, part_device=device,
                                 part_row0=self.row0)
        # kernels and the halo transport must share one stream (no host syncs)
        import torch
        self.torus.set_stream(torch.cuda.current_stream(device).cuda_stream)
        # packed edge rows: send top / bottom, receive top / bottom halo
        self.edges = [torch.empty(HALO * cols, dtype=torch.uint8, device=f"cuda:{device}")
                      for _ in range(4)]
        aligned = cols % 128 == 0 and all(
            slab_rows(global_rows, world, k)[1] % 32 == 0 and slab_rows(global_rows, world, k)[1] >= 32
            for k in range(world))
        self.ring = aligned if ring is None else (ring and aligned)
        if self.ring:
            handles = self.torus.ring_export()
            table = [(rank, self.rows, handles)]
            if world > 1:
                table = [None] * world
                self.dist.all_gather_object(table, (rank, self.rows, handles))
            by_rank = {r: (rows, h) for r, rows, h in table}
            up_rows, up_h = by_rank[self.plan.up]
            down_rows, down_h = by_rank[self.plan.down]
            ok = True
            try:  # needs peer access between the GPUs (NVLink / NVSwitch)
                self.torus.ring_connect(up_h, up_rows, down_h, down_rows)
            except Exception:  # noqa: BLE001 -- any failure: everyone falls back
                ok = False
            if world > 1:
                votes = [None] * world
                self.dist.all_gather_object(votes, ok)
                ok = all(votes)
            if not ok:
                self.torus.ring_disconnect()
                self.ring = False
        # Multi-generation (persistent) ring launches wait on the neighbours'
        # per-unit counters, which only persistent launches publish: every
        # rank must make the same choice, so it is voted on once here.
        self.persist = self.ring and self.torus.persistent_ok()
        if self.ring and world > 1:
            votes = [None] * world
            self.dist.all_gather_object(votes, self.persist)
            self.persist = all(votes)

    def use_stream(self, stream_ptr: int) -> None:
        self.torus.set_stream(stream_ptr)

    def _ring_fill(self) -> None:
        # every rank's interior must be in place and its kernels done before
        # the counters restart, and every rank's counters restarted before
        # anyone steps
        self.torus.synchronize()
        if self.plan.world > 1:
            self.dist.barrier()
        self.torus.ring_fill()
        self.torus.synchronize()
        if self.plan.world > 1:
            self.dist.barrier()

    def exchange(self) -> None:
        if self.ring:
            self._ring_fill()
            return
        send_top, send_bot, recv_top, recv_bot = self.edges
        self.torus.pack_edges(send_top.data_ptr(), send_bot.data_ptr())
        exchange_edges(send_top, send_bot, recv_top, recv_bot, self.plan, self.dist)
        self.torus.unpack_halo(recv_top.data_ptr(), recv_bot.data_ptr())

    def upload(self, interior) -> None:
        self.torus.upload(interior)
        self.exchange()

    def init_random(self, density: float, seed: int) -> None:
        self.torus.init_random(density, seed)
        self.exchange()

    def run(self, rule, steps: int) -> None:
        """`steps` generations, enqueued on the slab's stream.  On the ring
        every rank's kernel reads its neighbours' rows itself, so all steps go
        in one call (one persistent launch when the geometry allows it, the
        same decision on every rank: equal slab heights, neighbours on other
        GPUs); otherwise one step + packed exchange per generation."""
        if self.ring and self.persist:
            self.torus.run_async(rule, steps)
            return
        for _ in range(steps):  # one generation per launch on every rank
            self.step(rule)

    def step(self, rule, stencil: bool = False) -> None:
        if self.ring:
            if stencil:
                raise ValueError("config error: the stencil engine needs ring=False "
                                 "(padded halo rows)")
            self.torus.step_part(rule)  # the exchange happens inside the step
            return
        self.torus.step_part(rule, stencil=stencil)
        self.exchange()
