"""CPU, world_size 2 over gloo: the multi-GPU sharding host logic (row plan, record gather
to rank 0, stats reduction) reassembles exactly the 1-process encode.  The per-rank compute
is the oracle standing in for the GPU (the CUDA path is covered by test_gpu_encode)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1404_0774_b200.sharding import plan_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plan_rows():
    assert plan_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert plan_rows(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for rows in (1, 7, 64, 256):
        for world in (1, 2, 3, 8):
            p = plan_rows(rows, world)
            assert p[0][0] == 0 and p[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(p, p[1:]))


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
    import torch.distributed as dist

    import paper_1404_0774_b200 as fic
    from oracle import Oracle
    from paper_1404_0774_b200.sharding import encode_sharded, encode_volume_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    params = fic.CodecParams(n=4, step=4)

    def oracle_rows(img, b, e, p):
        R = img.shape[1] // p.n
        xs = np.tile(np.arange(R, dtype=np.int32) * p.n, e - b)
        ys = np.repeat(np.arange(b, e, dtype=np.int32) * p.n, R)
        return O.encode_ranges(img, dict(n=p.n, step=p.step), xs, ys)

    def oracle_batch(vol, p):
        encs, tot = [], {"candidates_tested": 0, "shadow_ranges": 0, "shadow_codeblocks": 0}
        for sl in vol:
            m, s = O.encode(sl, dict(n=p.n, step=p.step))
            encs.append(fic.EncodedImage(sl.shape[1], sl.shape[0], p, m))
            tot = {k: tot[k] + s[k] for k in tot}
        return encs, tot

    img = O.smooth_image(64, 77)
    enc = encode_sharded(img, params, encode_rows=oracle_rows)
    vol = np.stack([O.noise_image(32, 900 + i) for i in range(3)])
    encs, vstats = encode_volume_sharded(vol, params, encode_batch=oracle_batch)
    if rank == 0:
        q.put((enc.mappings.copy(), enc.stats, [e.mappings.copy() for e in encs], vstats))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gather_matches_single_process(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    maps, stats, vmaps, vstats = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want, wst = oracle.encode(oracle.smooth_image(64, 77), dict(n=4, step=4))
    assert np.array_equal(maps, want) and stats == wst
    total = 0
    for i in range(3):
        w, s = oracle.encode(oracle.noise_image(32, 900 + i), dict(n=4, step=4))
        assert np.array_equal(vmaps[i], w)
        total += s["candidates_tested"]
    assert vstats["candidates_tested"] == total
