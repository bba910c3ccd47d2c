"""Two processes on one GPU (gloo for the exchange: NCCL needs one device per rank) through
the real C-ABI shard entries: range-row shards of one image (fic_encode_rows and the
device-resident fic_encode_rows_device, SURVEY §8e / encoder.cpp:368-427's range-chunk split)
and slice shards of a volume, gathered to rank 0, equal the 1-process encode byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_1404_0774_b200 as fic
    from paper_1404_0774_b200 import images
    from paper_1404_0774_b200.abi import MAPPING_DTYPE
    from paper_1404_0774_b200.sharding import encode_sharded, encode_sharded_device, encode_volume_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    fic.set_device(0)
    params = fic.CodecParams(n=8, step=4)
    img = images.ct_slice(512, 1404002)
    host = encode_sharded(img, params)
    d_img = torch.from_numpy(img).cuda()
    dev, dstats = encode_sharded_device(d_img, 512, 512, params)
    vol = images.volume_slices(0, 3, 512)
    encs, vstats = encode_volume_sharded(vol, params)
    if rank == 0:
        q.put((host.mappings.copy(), host.stats, dev.cpu().numpy().view(MAPPING_DTYPE).copy(), dstats,
               [e.mappings.copy() for e in encs], vstats))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_one_gpu_match_single_process():
    import paper_1404_0774_b200 as fic
    from paper_1404_0774_b200 import images
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    maps, stats, dmaps, dstats, vmaps, vstats = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    params = fic.CodecParams(n=8, step=4)
    one = fic.encode(images.ct_slice(512, 1404002), params)
    assert one.mappings.tobytes() == maps.tobytes() == dmaps.tobytes()
    assert stats == dstats == one.stats
    total = 0
    for i, sl in enumerate(images.volume_slices(0, 3, 512)):
        e = fic.encode(sl, params)
        assert e.mappings.tobytes() == vmaps[i].tobytes()
        total += e.stats["candidates_tested"]
    assert vstats["candidates_tested"] == total
