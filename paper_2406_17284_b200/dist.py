"""Row-slab partitioning of one torus across processes (one per GPU).

Rank k of W owns global rows [k*R, (k+1)*R) with all columns.
One generation = the fused step kernel on every rank (ltl_step_part: main
kernel + local column wrap), then the only exchange the stencil needs: the
16 boundary rows of each slab go to the ring neighbours' halos

    my interior rows [16, 32)        -> rank-1's bottom halo rows [R+16, R+32)
    my interior rows [R, R+16)       -> rank+1's top halo rows    [0, 16)

as full padded-width rows (their column halos already refreshed), over NCCL
send/recv on the same stream as the kernels -- no host synchronisation.  The
same plan drives CPU tensors over gloo in the world-size-2 tests.
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


def exchange_rows(buf, pitch: int, rows: int, plan: HaloPlan, dist_mod=None) -> None:
    """Fill the 16 halo rows above / below a slab from its ring neighbours.

    buf: flat tensor (CUDA for NCCL, CPU for gloo) of (rows + 32) * pitch bytes
    holding the padded slab, interior rows at [16, 16 + rows).
    """
    if dist_mod is None:
        import torch.distributed as dist_mod  # noqa: N813
    band = HALO * pitch
    top_send = buf[HALO * pitch: HALO * pitch + band]
    bot_send = buf[rows * pitch: rows * pitch + band]
    top_recv = buf[0: band]
    bot_recv = buf[(rows + HALO) * pitch: (rows + HALO) * pitch + band]
    if plan.world == 1:
        top_recv.copy_(bot_send)
        bot_recv.copy_(top_send)
        return
    ops = [
        dist_mod.P2POp(dist_mod.isend, top_send, plan.up),
        dist_mod.P2POp(dist_mod.irecv, bot_recv, plan.down),
        dist_mod.P2POp(dist_mod.isend, bot_send, plan.down),
        dist_mod.P2POp(dist_mod.irecv, top_recv, plan.up),
    ]
    # With world == 2 both neighbours are the same rank; messages between a
    # pair match in issue order, and every rank issues (top, bottom) sends and
    # (bottom, top) receives, which pairs my top rows with the peer's bottom
    # halo and vice versa.
    for req in dist_mod.batch_isend_irecv(ops):
        req.wait()


class _CudaArray:
    """Zero-copy torch view of a device allocation owned by libltl_b200."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
            "strides": None,
        }


def slab_tensor(torus, which: int = 0):
    """torch.uint8 CUDA tensor aliasing the current padded slab buffer."""
    import torch
    ptr, pitch, rows = torus.slab_buffer(0, which)
    t = torch.as_tensor(_CudaArray(ptr, (rows + 2 * HALO) * pitch), device="cuda")
    return t, pitch, rows


class PartitionedTorus:
    """One rank's slab of a torus split across processes, driven through the C-ABI."""

    def __init__(self, global_rows: int, cols: int, rank: int, world: int, device: int):
        from .ltl import DeviceTorus
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

    def use_stream(self, stream_ptr: int) -> None:
        self.torus.set_stream(stream_ptr)

    def exchange(self) -> None:
        buf, pitch, rows = slab_tensor(self.torus)
        exchange_rows(buf, pitch, rows, self.plan)

    def init_random(self, density: float, seed: int) -> None:
        self.torus.init_random(density, seed)
        self.exchange()

    def step(self, rule, stencil: bool = False) -> None:
        self.torus.step_part(rule, stencil=stencil)
        self.exchange()
