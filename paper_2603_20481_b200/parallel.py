"""Multi-GPU plumbing for the capture-sharded path.

TF plots (captures) are independent, so the work shards by capture with no
data-path collective.  The one exchange step is collecting the detections on
rank 0: each rank sends its per-plot box counts, then only the boxes those
counts say exist (count-prefixed records, ~32 B per box), over point-to-point
send/recv -- NCCL on CUDA tensors (bench.py), gloo on CPU tensors (tests).
bench.py calls exactly these functions inside its timed step.
"""
from __future__ import annotations


def capture_shard(total: int, rank: int, world: int) -> range:
    """Contiguous balanced shard of `total` captures for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def pack_detections(n_boxes, boxes):
    """(P,) int32 counts + (P, K, 4) fixed-capacity records -> (counts clamped to
    K, (sum counts, 4) packed records in plot order), on the records' device."""
    import torch

    K = boxes.shape[1]
    counts = n_boxes.clamp(max=K)
    mask = torch.arange(K, device=boxes.device)[None, :] < counts[:, None]
    return counts, boxes[mask]


def gather_detections(n_boxes, boxes, group=None, root: int = 0):
    """Collect every rank's detections on `root`.

    Each rank sends its counts (P,) then its packed records (sum counts, 4);
    root returns [(counts, packed)] per rank in rank order (its own included),
    the other ranks return None.  P and K may differ between ranks."""
    import torch
    import torch.distributed as dist

    counts, packed = pack_detections(n_boxes, boxes)
    counts = counts.contiguous()
    packed = packed.contiguous()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if rank != root:
        meta = torch.tensor([counts.numel()], dtype=torch.int64, device=counts.device)
        dist.send(meta, dst=root, group=group)
        dist.send(counts, dst=root, group=group)
        if packed.numel():
            dist.send(packed, dst=root, group=group)
        return None
    out = []
    for r in range(world):
        if r == root:
            out.append((counts, packed))
            continue
        meta = torch.empty(1, dtype=torch.int64, device=counts.device)
        dist.recv(meta, src=r, group=group)
        c = torch.empty(int(meta.item()), dtype=counts.dtype, device=counts.device)
        dist.recv(c, src=r, group=group)
        n = int(c.sum().item())
        p = torch.empty((n, 4), dtype=packed.dtype, device=packed.device)
        if n:
            dist.recv(p, src=r, group=group)
        out.append((c, p))
    return out


def flatten_detections(gathered) -> list:
    """Root's gather result -> per-capture list of (n, 4) numpy boxes in global
    capture order (rank-major: rank r holds captures capture_shard(r))."""
    out = []
    for counts, packed in gathered:
        c = counts.cpu().tolist()
        p = packed.cpu().numpy()
        o = 0
        for n in c:
            out.append(p[o:o + n])
            o += n
    return out
