"""Multi-GPU encode by range sharding: one process per GPU.

* single image (cfg4): the range grid's rows are split into contiguous blocks, one per
  rank; every rank builds the full domain pool from its own copy of the image (the pool
  is replicated: cheaper to rebuild than to exchange) and encodes only its rows through
  the C-ABI (fic_encode_rows); the fixed-size 32-byte code records are gathered to rank 0.
* volume (cfg5): slices are split into contiguous blocks per rank, each encoded whole.

Ranges are independent, so the records are byte-identical to a 1-GPU encode for every
world size (the invariant of proj/tests/acceptance.cpp:49-69).  The gather is the only
exchange; it uses torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
import numpy as np

from .abi import MAPPING_DTYPE


def plan_rows(rows, world):
    """Contiguous [begin, end) row blocks, sizes differing by at most one."""
    base, extra = divmod(rows, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def _gather_records(recs, counts, group, device):
    """Gather variable-length record arrays to rank 0 (padded to the max count)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    maxc = max(counts)
    buf = np.zeros(maxc, MAPPING_DTYPE)
    buf[: len(recs)] = recs
    t = torch.from_numpy(buf.view(np.uint8).copy()).to(device)
    out = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gather_list=out, dst=0, group=group)
    if rank != 0:
        return None
    parts = [out[r].cpu().numpy().view(MAPPING_DTYPE)[: counts[r]] for r in range(world)]
    return np.concatenate(parts) if parts else np.zeros(0, MAPPING_DTYPE)


def _sum_stats(stats, group, device):
    import torch
    import torch.distributed as dist
    t = torch.tensor([stats["candidates_tested"], stats["shadow_ranges"], stats["shadow_codeblocks"]],
                     dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    v = t.cpu().tolist()
    return {"candidates_tested": v[0], "shadow_ranges": v[1], "shadow_codeblocks": v[2]}


def encode_sharded(image, params, group=None, device="cpu", encode_rows=None):
    """Range-sharded encode of one image.  Every rank passes the same image; rank 0 gets
    the full EncodedImage (others get None).  `encode_rows(image, begin, end, params)`
    returns (records, stats) for range rows [begin, end); default: the C-ABI path."""
    import torch.distributed as dist

    from . import codec
    encode_rows = encode_rows or codec.encode_rows
    img = np.ascontiguousarray(image, np.uint8)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    rows = img.shape[0] // params.n
    plan = plan_rows(rows, world)
    b, e = plan[rank]
    recs, st = encode_rows(img, b, e, params)
    counts = [(pe - pb) * (img.shape[1] // params.n) for pb, pe in plan]
    full = _gather_records(recs, counts, group, device)
    stats = _sum_stats(st, group, device)
    if rank != 0:
        return None
    return codec.EncodedImage(img.shape[1], img.shape[0], params, full, stats)


def encode_volume_sharded(volume, params, group=None, device="cpu", encode_batch=None):
    """Slice-sharded encode of a (count, side, side) volume; rank 0 gets the list of
    EncodedImage in slice order.  `encode_batch(slices, params)` -> (encs, stats)."""
    import torch.distributed as dist

    from . import codec
    encode_batch = encode_batch or codec.encode_batch
    vol = np.ascontiguousarray(volume, np.uint8)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    plan = plan_rows(vol.shape[0], world)
    b, e = plan[rank]
    per = (vol.shape[1] // params.n) * (vol.shape[2] // params.n)
    if e > b:
        encs, st = encode_batch(vol[b:e], params)
        recs = np.concatenate([x.mappings for x in encs])
    else:
        recs = np.zeros(0, MAPPING_DTYPE)
        st = {"candidates_tested": 0, "shadow_ranges": 0, "shadow_codeblocks": 0}
    counts = [(pe - pb) * per for pb, pe in plan]
    full = _gather_records(recs, counts, group, device)
    stats = _sum_stats(st, group, device)
    if rank != 0:
        return None, stats
    return [codec.EncodedImage(vol.shape[2], vol.shape[1], params, full[i * per:(i + 1) * per].copy())
            for i in range(vol.shape[0])], stats


def encode_sharded_device(d_image, width, height, params, group=None, stream=None):
    """Range-sharded encode of one device-resident image (torch uint8 tensor, every rank holds
    the whole image): rank r encodes its block of range rows into device records
    (fic_encode_rows_device, a replicated pool per GPU) and the records are gathered to rank 0
    over the process group (NCCL: NVLink on one box).  Rank 0 gets a (ranges x 32) uint8
    device tensor of every record in range order; all ranks get the summed stats."""
    import torch
    import torch.distributed as dist

    from . import codec
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    rows = height // params.n
    rx = width // params.n
    plan = plan_rows(rows, world)
    b, e = plan[rank]
    maxc = max(pe - pb for pb, pe in plan) * rx
    shard = torch.zeros(maxc * 32, dtype=torch.uint8, device=d_image.device)
    st_handle = stream if stream is not None else torch.cuda.current_stream(d_image.device).cuda_stream
    st = codec.encode_rows_device(d_image.data_ptr(), width, height, b, e, shard.data_ptr(), params, st_handle)
    if dist.get_backend(group) != "nccl":  # gloo (tests: several ranks on one GPU) gathers host tensors
        shard = shard.cpu()
    out = [torch.empty_like(shard) for _ in range(world)] if rank == 0 else None
    dist.gather(shard, gather_list=out, dst=0, group=group)
    stats = _sum_stats(st, group, shard.device)
    if rank != 0:
        return None, stats
    full = torch.cat([out[r][: (pe - pb) * rx * 32] for r, (pb, pe) in enumerate(plan)])
    return full, stats
