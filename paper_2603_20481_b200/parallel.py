"""Multi-GPU plumbing for the capture-sharded path.

TF plots (captures) are independent, so the work shards by capture with no
data-path collective; the one exchange step is gathering each rank's
fixed-capacity detection records (n_boxes per plot + box records) so every
rank -- rank 0 in particular -- holds the whole job's detections.  Works with
NCCL on CUDA tensors (bench.py) and gloo on CPU tensors (tests)."""
from __future__ import annotations


def capture_shard(total: int, rank: int, world: int) -> range:
    """Contiguous balanced shard of `total` captures for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_detections(n_boxes, boxes, group=None):
    """all_gather of per-plot box counts (P,) int32 and records (P, K, 4) f64.

    Returns (counts (world, P), records (world, P, K, 4)) on every rank; all
    ranks must pass the same P and K (fixed capacity keeps one collective)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = torch.empty((world,) + tuple(n_boxes.shape), dtype=n_boxes.dtype, device=n_boxes.device)
    recs = torch.empty((world,) + tuple(boxes.shape), dtype=boxes.dtype, device=boxes.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(counts, n_boxes.contiguous(), group=group)
        dist.all_gather_into_tensor(recs, boxes.contiguous(), group=group)
    else:
        dist.all_gather(list(counts.unbind(0)), n_boxes.contiguous(), group=group)
        dist.all_gather(list(recs.unbind(0)), boxes.contiguous(), group=group)
    return counts, recs


def flatten_detections(counts, recs) -> list:
    """(world, P[, K, 4]) gathered tensors -> per-capture list of (n, 4) boxes in
    global capture order (rank-major: rank r holds captures capture_shard(r))."""
    out = []
    for r in range(counts.shape[0]):
        for p in range(counts.shape[1]):
            n = int(counts[r, p])
            out.append(recs[r, p, :n].cpu().numpy())
    return out
