"""Multi-GPU partitioning of the hot path.

The reference's only parallelism is a thread pool over fixed 96-row bands
with halos (parallel.py:43-66, kernels.py:152-153) and a bit-identical-for-any-
thread-count contract (parallel.py:1-10).  Here one process drives one GPU
(``torch.distributed``, NCCL over NVLink on a GPU box, gloo in the CPU tests)
and the same contract holds across GPU counts:

* **frame batch** (C3/C4): frames ``shard_range(B, rank, world)`` per rank, no
  collective in the data path.  Exact integer-weighted fp64 sums make every
  output independent of the partition.
* **strip partition** (C5, one very large frame): rank g owns rows
  ``StripPlan.owned(g)``; it needs ``halo`` rows of its neighbours (the fit's
  radius, >= 1 for the depth-Laplacian predicate), exchanged with grouped
  P2P send/recv (``exchange_halo``) or sliced from the host frame at upload.
  Each rank runs the fused pass on its extended block and keeps its owned
  rows; labels are computed on the owned rows (predicate on the extended
  block) with global raster indices, then merged across the seams:
  every rank contributes its first and last owned label rows to one
  all-gather (2 x W int32 per rank, into device memory), runs the same
  deterministic min-root union-find over them on its device
  (``sn_seam_merge``: no host round trip) and remaps its labels there
  (``sn_relabel_table``).  That gather is the only collective of the path.
  (``sn_seam_merge_host`` is the same merge on the host, used by the CPU
  tests.)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced share [start, stop) of ``n`` items for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n), world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class StripPlan:
    """Row partition of one H x W frame into ``n_strips`` strips with a halo.

    ``halo`` = max(fit radius, 1): the fit reads R rows either side
    (kernels.py:153) and the depth Laplacian one (adaptive.py:80-97)."""

    height: int
    width: int
    n_strips: int
    halo: int

    @classmethod
    def for_kernel(cls, height: int, width: int, n_strips: int, kernel_size: int = 9):
        return cls(int(height), int(width), int(n_strips), max(int(kernel_size) // 2, 1))

    def __post_init__(self):
        if self.n_strips < 1 or self.height < self.n_strips:
            raise ValueError("need 1 <= n_strips <= height")
        if self.halo < 1:
            raise ValueError("halo must be >= 1")
        if min(b - a for a, b in (self.owned(s) for s in range(self.n_strips))) < self.halo:
            raise ValueError("every strip must own at least `halo` rows")

    def owned(self, s: int) -> tuple[int, int]:
        return shard_range(self.height, s, self.n_strips)

    def block(self, s: int) -> tuple[int, int]:
        """Rows [b0, b1) the strip's kernels read: owned rows + halo, clipped."""
        r0, r1 = self.owned(s)
        return max(0, r0 - self.halo), min(self.height, r1 + self.halo)

    def owned_in_block(self, s: int) -> tuple[int, int]:
        r0, r1 = self.owned(s)
        b0, _ = self.block(s)
        return r0 - b0, r1 - b0


# ---------------------------------------------------------------------------
# collectives (torch.distributed; tensors on the group's device)


def exchange_halo(owned, plan: StripPlan, rank: int, group=None):
    """Build the extended block ``plan.block(rank)`` from this rank's owned
    rows ``owned`` ([rows, W]) and its neighbours' edge rows, exchanged with
    one grouped P2P round (NCCL send/recv over NVLink; gloo on CPU)."""
    import torch
    import torch.distributed as dist

    h = plan.halo
    r0, r1 = plan.owned(rank)
    if owned.shape[0] != r1 - r0:
        raise ValueError("owned rows do not match the plan")
    b0, b1 = plan.block(rank)
    block = torch.empty((b1 - b0,) + tuple(owned.shape[1:]), dtype=owned.dtype,
                        device=owned.device)
    top, bot = r0 - b0, r1 - b0
    block[top:bot] = owned
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, owned[:h].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, block[:top], rank - 1, group))
    if rank + 1 < plan.n_strips:
        ops.append(dist.P2POp(dist.isend, owned[-h:].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, block[bot:], rank + 1, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return block


def gather_seams_device(labels_owned, world: int, group=None):
    """All-gather every rank's first and last owned label rows into one int32
    ``[world, 2, W]`` tensor on this rank's device (NCCL over NVLink on a GPU
    box), identical on every rank."""
    import torch
    import torch.distributed as dist

    edge = torch.stack([labels_owned[0], labels_owned[-1]]).to(torch.int32).contiguous()
    if not edge.is_cuda:  # gloo (the CPU tests): the list form
        parts = [torch.empty_like(edge) for _ in range(world)]
        dist.all_gather(parts, edge, group=group)
        return torch.stack(parts)
    out = torch.empty((world,) + tuple(edge.shape), dtype=torch.int32, device=edge.device)
    dist.all_gather_into_tensor(out, edge, group=group)
    return out


def gather_seams(labels_owned, world: int, group=None) -> np.ndarray:
    """The gathered seam rows on the host (int32 ``[world, 2, W]``)."""
    return gather_seams_device(labels_owned, world, group).cpu().numpy()


def seam_map(labels_owned, world: int, group=None) -> tuple[np.ndarray, np.ndarray]:
    """Collective + deterministic host merge: (label -> root) pairs of every
    label that changes, sorted by label, identical on every rank."""
    from .device import seam_merge

    return seam_merge(gather_seams(labels_owned, world, group))


# ---------------------------------------------------------------------------
# per-rank device work


def strip_pass(block, plan: StripPlan, s: int, rig, kernels=9, threshold: float = 0.2):
    """Fused pass over the strip's extended block (fit + normal + point + the
    passable bits in one read), then labels of the owned rows from the bits
    with global raster indices (before the seam merge).  Returns views of the
    owned rows: (points ``[rows, W, 6]``, labels ``[rows, W]``) -- identical to
    the same rows of the whole-frame result, because the owned rows are at
    least ``halo`` rows from any block edge that is not an image edge."""
    from . import device

    o0, o1 = plan.owned_in_block(s)
    b0, _ = plan.block(s)
    r0, _ = plan.owned(s)
    pts, bits = device.oriented_points_bits(block, rig, kernels, threshold, row0=b0)
    lab = device.labels_from_bits(bits[:, o0:o1].contiguous(), plan.width, row_base=r0)
    return pts[0, o0:o1], lab[0]


def apply_seam_map(labels, plan: StripPlan, s: int, keys: np.ndarray, vals: np.ndarray):
    """Remap one strip's labels in place on its device."""
    import torch
    from . import device

    dev = labels.device
    r0, _ = plan.owned(s)
    n = max(1, len(keys))
    k = torch.full((n,), -1, dtype=torch.int32)
    v = torch.full((n,), -1, dtype=torch.int32)
    k[:len(keys)] = torch.from_numpy(np.asarray(keys, dtype=np.int32))
    v[:len(vals)] = torch.from_numpy(np.asarray(vals, dtype=np.int32))
    nm = torch.tensor([len(keys)], dtype=torch.int32)
    return device.relabel(labels, k.to(dev), v.to(dev), nm.to(dev), r0 * plan.width)


def distributed_strip_frame(owned, plan: StripPlan, rig, kernels=9, threshold: float = 0.2,
                            group=None):
    """One rank's share of a strip-partitioned frame: halo exchange, fused
    pass, labels, seam merge.  Returns (points [rows, W, 6], labels [rows, W])
    for the owned rows -- bit-identical to the whole-frame result."""
    import torch.distributed as dist

    from . import device

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world != plan.n_strips:
        raise ValueError("one strip per rank")
    block = exchange_halo(owned, plan, rank, group)
    pts, lab = strip_pass(block, plan, rank, rig, kernels, threshold)
    if lab.is_cuda:
        # the merge on the device: all-gather, min-root union-find over the
        # seams, relabel -- no host round trip
        seams = gather_seams_device(lab, world, group)
        device.relabel_table(lab, device.seam_table(seams, plan.height * plan.width))
    else:  # CPU tensors (gloo tests): the host merge
        keys, vals = seam_map(lab, world, group)
        apply_seam_map(lab, plan, rank, keys, vals)
    return pts, lab


def local_strip_frame(disp, plan: StripPlan, rig, kernels=9, threshold: float = 0.2):
    """All strips of one frame on ONE device, in sequence (no cross-strip
    waiting): exercises the strip path -- block slicing, per-strip passes,
    seam merge, relabel -- against the whole-frame result on a single GPU."""
    import torch

    if disp.dim() != 2:
        raise ValueError("disp must be one [H, W] frame")
    pts, labs = [], []
    for s in range(plan.n_strips):
        b0, b1 = plan.block(s)
        p_s, l_s = strip_pass(disp[b0:b1].contiguous(), plan, s, rig, kernels, threshold)
        pts.append(p_s)
        labs.append(l_s)
    from . import device
    seams = torch.stack([torch.stack([lab[0], lab[-1]]) for lab in labs]).to(torch.int32)
    table = device.seam_table(seams, plan.height * plan.width)
    for lab in labs:
        device.relabel_table(lab, table)
    return torch.cat(pts), torch.cat(labs)
