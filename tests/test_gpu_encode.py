"""GPU parity of the encoder: libfic_b200 (through its C-ABI) against the oracle.

Bar (north_star): emitted codes identical to the reference, residuals bit-equal
(proj/tests/oracle.hpp:140-143 demands exact residual bits), EncodeStats identical.
Both matchers are checked: the tcgen05 matcher (default for n in {2,4,8}) and the
CUDA-core matcher (FIC_MATCHER=simt, the parity anchor and the n >= 16 path).
"""
import os

import numpy as np
import pytest

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import images

pytestmark = pytest.mark.gpu

KEYS = ["x", "y", "sym", "qs", "qo"]


def assert_same(got, want, ctx=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, ctx
    for k in KEYS:
        bad = np.nonzero(got[k] != want[k])[0]
        assert len(bad) == 0, f"{ctx}: field {k} differs at ranges {bad[:10]}: got {got[bad[:3]]} want {want[bad[:3]]}"
    # residual bits
    gb = got["residual"].view(np.uint64)
    wb = want["residual"].view(np.uint64)
    bad = np.nonzero(gb != wb)[0]
    assert len(bad) == 0, f"{ctx}: residual bits differ at {bad[:10]}: {got['residual'][bad[:3]]} vs {want['residual'][bad[:3]]}"


class env:
    """Temporarily set environment variables (the library reads them on every call)."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = os.environ.get(k)
            os.environ[k] = str(v)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


# "tc": the tcgen05 scan (default), "simt": the CUDA-core matcher (parity anchor, n >= 16 path)
MATCHERS = {"tc": dict(FIC_MATCHER="tc"), "simt": dict(FIC_MATCHER="simt")}


@pytest.fixture(params=list(MATCHERS))
def matcher(request):
    with env(**MATCHERS[request.param]):
        yield request.param


VARIANTS = [dict(), dict(step=2, s_max=0.75), dict(o_bits=6, s_bits=4)]


@pytest.mark.parametrize("vi", range(3))
def test_noise32_oracle_variants(oracle, matcher, vi):
    # test_encoder.cpp:152-167: noise_image(32, 50..52) x three parameter variants
    pv = VARIANTS[vi]
    img = oracle.noise_image(32, 50 + vi)
    enc = fic.encode(img, fic.CodecParams(**pv))
    want, st = oracle.encode(img, pv)
    assert_same(enc.mappings, want, f"noise32 {pv}")
    assert enc.stats == st


@pytest.mark.parametrize("seed", [201, 202, 203, 204, 205])
def test_acceptance_oracle_optimality(oracle, matcher, seed):
    # acceptance.cpp:73-91
    img = oracle.noise_image(32, seed)
    enc = fic.encode(img)
    want, _ = oracle.encode(img, {}, brute=True)
    assert_same(enc.mappings, want, f"noise32 seed {seed}")


@pytest.mark.parametrize("n,step", [(2, 1), (2, 2), (4, 1), (4, 3), (8, 1), (8, 3), (8, 8), (16, 4), (16, 16)])
def test_geometries_smooth_and_noise(oracle, matcher, n, step):
    side = max(64, 4 * n)
    for img in (oracle.smooth_image(side, 52 + n), oracle.noise_image(side, 7 + step)):
        pv = dict(n=n, step=step)
        enc = fic.encode(img, fic.CodecParams(**pv))
        want, st = oracle.encode(img, pv)
        assert_same(enc.mappings, want, f"n={n} step={step}")
        assert enc.stats == st


def test_shadow_and_flat(oracle, matcher):
    # constant image: every range is a shadow (test_encoder.cpp:102-121)
    for v in (0, 128, 255):
        img = np.full((16, 16), v, np.uint8)
        enc = fic.encode(img)
        want, st = oracle.encode(img, {})
        assert_same(enc.mappings, want, f"constant {v}")
        assert enc.stats == st and st["shadow_ranges"] == 16 and st["candidates_tested"] == 0
    # flat-codebook fallback (test_encoder.cpp:243-258)
    img = np.full((32, 32), 100, np.uint8)
    for y in range(32):
        for x in range(28, 32):
            img[y, x] = ((x + y) % 2) * 255
    rec, st = fic.encode_range(img, 28, 0, fic.CodecParams(step=5))
    want, wst = oracle.encode_ranges(img, dict(step=5), [28], [0])
    assert_same(np.array([rec]), want)
    assert st == wst and st["candidates_tested"] == 0 and st["shadow_codeblocks"] > 0
    # partly flat image with shadow_eps > 0
    img = oracle.smooth_image(64, 5)
    img[:, :24] = 77
    for pv in (dict(), dict(shadow_eps=40.0), dict(n=8, step=2, shadow_eps=500.0)):
        enc = fic.encode(img, fic.CodecParams(**pv))
        want, st = oracle.encode(img, pv)
        assert_same(enc.mappings, want, f"flat {pv}")
        assert enc.stats == st


def test_constructed_exact_match(oracle, matcher):
    # test_encoder.cpp:131-150
    rng_pattern = oracle.mt19937(43, 16) % 256
    img = oracle.noise_image(16, 44)
    for r in range(8):
        for c in range(8):
            img[r, c] = rng_pattern[(r // 2) * 4 + c // 2]
    for r in range(4):
        for c in range(4):
            img[8 + r, 8 + c] = rng_pattern[r * 4 + c]
    rec, _ = fic.encode_range(img, 8, 8)
    assert rec["residual"] == 0.0
    want, _ = oracle.encode_ranges(img, {}, [8], [8])
    assert_same(np.array([rec]), want)


def test_cfg1_phantom_full(oracle, matcher):
    img = images.phantom(256, 1404001)
    pv = dict(n=8, step=8)
    enc = fic.encode(img, fic.CodecParams(**pv))
    want, st = oracle.encode_threaded(img, pv)
    assert_same(enc.mappings, want, "cfg1")
    assert enc.stats == st


def test_cfg2_ct_slice_full(oracle):
    img = images.ct_slice(512, 1404002)
    pv = dict(n=8, step=4)
    enc = fic.encode(img, fic.CodecParams(**pv))
    want, st = oracle.encode_threaded(img, pv)
    assert_same(enc.mappings, want, "cfg2")
    assert enc.stats == st


def test_cfg2_full_vs_compiled_reference():
    """cfg2 in full against the unmodified reference itself (oracle/_ref: its encode_parallel,
    proj/src/encoder.cpp:368-427, over every host thread): records, residual bits, stats."""
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    img = images.ct_slice(512, 1404002)
    pv = dict(n=8, step=4)
    want, st = Reference().encode(img, pv, workers=os.cpu_count() or 1)
    enc = fic.encode(img, fic.CodecParams(**pv))
    assert_same(enc.mappings, want, "cfg2 vs reference")
    assert enc.stats == st


def test_cfg3_full(oracle):
    """cfg3 (512x512, 4x4 ranges, domain stride 2) in full: all 16,384 ranges."""
    img = images.ct_slice(512, 1404002)
    pv = dict(n=4, step=2)
    enc = fic.encode(img, fic.CodecParams(**pv))
    want, st = oracle.encode_threaded(img, pv)
    assert_same(enc.mappings, want, "cfg3")
    assert enc.stats == st


def _oracle_rows_many(oracle, jobs, pv):
    """Oracle records of (image, range row) jobs, spread over every host thread."""
    from concurrent.futures import ThreadPoolExecutor
    n = pv["n"]

    def one(job):
        img, row = job
        RX = img.shape[1] // n
        xs = np.arange(RX, dtype=np.int32) * n
        ys = np.full(RX, row * n, np.int32)
        return oracle.encode_ranges(img, pv, xs, ys)[0]

    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        return list(ex.map(one, jobs))


def test_cfg5_as_benched(oracle):
    """cfg5 exactly as bench.py runs it: one stacked 64-slice pass of the benched volume
    (images.volume_slices, 512x512 CT slices, n=8, step 4) through fic_encode_batch_device.
    Every slice is checked against the oracle on 4 seeded-random range rows (rows 0 and 63
    included across the volume), and each slice's EncodeStats contribution against the
    oracle's domain pool flat count and the ranges' variances."""
    import torch
    from paper_1404_0774_b200.abi import MAPPING_DTYPE
    count, side, n = 64, 512, 8
    pv = dict(n=n, step=4)
    vol = images.volume_slices(0, count, 512)
    per = (side // n) ** 2
    d_img = torch.from_numpy(vol).cuda()
    d_out = torch.zeros(count * per * MAPPING_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    st = fic.encode_batch_device(d_img.data_ptr(), count, side, side, d_out.data_ptr(), fic.CodecParams(**pv))
    got = d_out.cpu().numpy().view(MAPPING_DTYPE).reshape(count, per)
    rng = np.random.default_rng(1404005)
    jobs, where = [], []
    for z in range(count):
        rows = rng.choice(64, 4, replace=False)
        if z == 0:
            rows[0] = 0
        if z == count - 1:
            rows[0] = 63
        for r in rows:
            jobs.append((vol[z], int(r)))
            where.append((z, int(r)))
    wants = _oracle_rows_many(oracle, jobs, pv)
    for (z, r), want in zip(where, wants):
        assert_same(got[z, r * 64:(r + 1) * 64], want, f"cfg5 slice {z} row {r}")
    # stats: candidates_tested = 8 (R - shadow)(D - flat) per slice (encoder.hpp:49-53)
    total = {"candidates_tested": 0, "shadow_ranges": 0, "shadow_codeblocks": 0}
    for z in range(count):
        _, _, _, flat = oracle.domain_pool(vol[z], pv)
        b = vol[z].astype(np.int64).reshape(64, n, 64, n).transpose(0, 2, 1, 3).reshape(per, n * n)
        shadow = int(np.sum(n * n * np.sum(b * b, 1) - np.sum(b, 1) ** 2 <= 0))
        D, F = len(flat), int(flat.sum())
        total["candidates_tested"] += 8 * (per - shadow) * (D - F)
        total["shadow_ranges"] += shadow
        total["shadow_codeblocks"] += 8 * (per - shadow) * F
    assert st == total


def test_cfg4_reference_rows():
    """cfg4 (2048x2048, n=8, step 2) on 16 full range rows (first, last and 14 seeded random;
    each includes the first and last columns) against the UNMODIFIED reference's records
    (tests/golden/cfg4_rows.npz, generated by tests/golden/make_cfg4_rows.py: ~37 s of reference
    search per row on 16 threads), with the default fp16 full level (scan mode 6), with it forced
    off (mode 1) and with fp16 hit-first sparse levels (mode 7 instead of 2)."""
    import hashlib
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg4_rows.npz")
    fx = np.load(path)
    img = images.xray(2048, 1404004)
    assert hashlib.sha256(img.tobytes()).digest() == fx["image_sha256"].tobytes()
    rows = [int(r) for r in fx["rows"]]
    want = fx["maps"]
    R = 2048 // 8
    for sw in (dict(), dict(FIC_F16ACC="0"), dict(FIC_F16SEL="1")):
        with env(**sw):
            enc = fic.encode(img, fic.CodecParams(n=8, step=2))
        got = np.concatenate([enc.mappings[r * R:(r + 1) * R] for r in rows])
        assert_same(got, want, f"cfg4 rows {sw}")


def test_parallel_api_and_rows(oracle):
    img = oracle.noise_image(64, 53)
    seq = fic.encode(img)
    par = fic.encode(img, workers=4, chunk=(8, 8))
    assert seq.serialize() == par.serialize()
    # range-row shards reassemble to the full encode (multi-GPU sharding unit)
    R = 64 // 4
    parts = [fic.encode_rows(img, a, b)[0] for a, b in [(0, 5), (5, 11), (11, 16)]]
    assert_same(np.concatenate(parts), seq.mappings, "rows")
    with pytest.raises(fic.CodecError, match="BadParams"):
        fic.encode(img, workers=2, chunk=(0, 4))
    with pytest.raises(fic.CodecError, match="GeometryError"):
        fic.encode_range(img, 3, 0)


def test_batch(oracle):
    vol = np.stack([oracle.noise_image(32, 300 + i) for i in range(3)])
    encs, st = fic.encode_batch(vol)
    total = 0
    for i in range(3):
        want, s = oracle.encode(vol[i], {})
        assert_same(encs[i].mappings, want, f"slice {i}")
        total += s["candidates_tested"]
    assert st["candidates_tested"] == total


@pytest.mark.parametrize("scan", ["tc"])
@pytest.mark.parametrize("pv,chunk", [(dict(n=4, step=2), "64"), (dict(n=8, step=3), "2"), (dict(n=2, step=1), "3")])
def test_batch_stacked(oracle, scan, pv, chunk):
    """Slices stacked into one encode pass (slice-offset pools, one scan over every slice's
    ranges): each slice's records and the summed stats equal the oracle's per-slice encode.
    Slices differ in content (noise, smooth, a constant slice, a half-flat slice) so flat
    domains and shadow ranges are counted per slice; chunk 2 and 3 leave a ragged last pass."""
    side = 64
    vol = np.stack([oracle.noise_image(side, 500 + i) for i in range(5)])
    vol[1] = oracle.smooth_image(side, 77)
    vol[2] = 123
    vol[3, :, : side // 2] = 40
    total = {"candidates_tested": 0, "shadow_ranges": 0, "shadow_codeblocks": 0}
    wants = []
    for i in range(len(vol)):
        want, st = oracle.encode(vol[i], pv)
        wants.append(want)
        for k in total:
            total[k] += st[k]
    with env(FIC_BATCH_CHUNK=chunk, **MATCHERS[scan]):
        encs, st = fic.encode_batch(vol, fic.CodecParams(**pv))
    for i, want in enumerate(wants):
        assert_same(encs[i].mappings, want, f"slice {i} {pv} chunk {chunk}")
    assert st == total


def test_batch_device_cfg5_shape(oracle):
    """fic_encode_batch_device on cfg5 slices (512x512 CT slices, n=8, step 4), three slices in
    one pass: every slice against fic_encode of that slice (itself oracle-checked by the cfg2
    test), and slice 2's first two range rows against the oracle directly."""
    import torch
    from paper_1404_0774_b200.abi import MAPPING_DTYPE
    vol = images.volume(count=3, side=512)
    p = fic.CodecParams(n=8, step=4)
    per = (512 // 8) ** 2
    d_img = torch.from_numpy(vol).cuda()
    d_out = torch.zeros(3 * per * MAPPING_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    st = fic.encode_batch_device(d_img.data_ptr(), 3, 512, 512, d_out.data_ptr(), p)
    got = d_out.cpu().numpy().view(MAPPING_DTYPE)
    total = 0
    for i in range(3):
        enc = fic.encode(vol[i], p)
        assert_same(got[i * per:(i + 1) * per], enc.mappings, f"slice {i}")
        total += enc.stats["candidates_tested"]
    assert st["candidates_tested"] == total
    rows, _ = oracle.encode_threaded(vol[2], {"n": 8, "step": 4}, rows=[0, 1])
    assert_same(got[2 * per:2 * per + len(rows)], rows, "slice 2 oracle rows")


@pytest.mark.parametrize("mode", ["exhaustive", "no_prepass", "tiny_list"])
def test_pruning_is_output_neutral(oracle, mode):
    """The scan's bound, the sparse levels and the survivor-list overflow path never change the
    result: exhaustive evaluation (every candidate through the exact path), a single full level,
    and a list so small that every level overflows and the full level is re-run all give the
    reference's records."""
    settings = {"exhaustive": dict(FIC_DEBUG=1), "no_prepass": dict(FIC_PREPASS=0),
                "tiny_list": dict(FIC_LIST_CAP=4096)}
    img = oracle.noise_image(64, 911)
    img[:16, :16] = 90  # some shadow ranges and flat domains
    for pv in (dict(n=4, step=1), dict(n=8, step=2), dict(n=2, step=3)):
        want, st = oracle.encode(img, pv)
        with env(**settings[mode]):
            enc = fic.encode(img, fic.CodecParams(**pv))
        assert_same(enc.mappings, want, f"{mode} {pv}")
        assert enc.stats == st


def test_graph_replay_new_contents(oracle):
    """Repeated encodes of one geometry run as a captured CUDA graph from the third call on;
    replays must follow new image contents, timing switches and list-capacity changes, and
    match the eager path (FIC_NO_GRAPH=1) and the oracle."""
    pv = dict(n=4, step=2)
    imgs = [oracle.noise_image(64, 70 + k) for k in range(2)] + [oracle.smooth_image(64, 71)]
    want = [oracle.encode(im, pv) for im in imgs]
    for rep in range(4):
        for k, im in enumerate(imgs):
            enc = fic.encode(im, fic.CodecParams(**pv))
            assert_same(enc.mappings, want[k][0], f"graph rep {rep} image {k}")
            assert enc.stats == want[k][1]
    fic.set_matcher_timing(True)
    try:
        for k, im in enumerate(imgs * 3):
            assert_same(fic.encode(im, fic.CodecParams(**pv)).mappings, want[k % 3][0], "timed graph")
        assert fic.matcher_timing(reset=True)[1] > 0
    finally:
        fic.set_matcher_timing(False)
    with env(FIC_LIST_CAP="300"):  # overflow: the full level re-runs eagerly with grown lists
        for k, im in enumerate(imgs * 2):
            assert_same(fic.encode(im, fic.CodecParams(**pv)).mappings, want[k % 3][0], "tiny list")
    with env(FIC_NO_GRAPH="1"):
        for k, im in enumerate(imgs):
            assert_same(fic.encode(im, fic.CodecParams(**pv)).mappings, want[k][0], "eager")


@pytest.mark.parametrize("coarse", ["0", "1"])
def test_coarse_vote_output_neutral(oracle, coarse):
    """The whole-tile |max| vote (default for pools above 1024 tiles) forced on and off on
    small images: identical codes and residual bits."""
    for img, pv in [(oracle.noise_image(64, 9), dict(n=4, step=2)), (oracle.smooth_image(64, 5), dict(n=8, step=2)),
                    (images.ct_slice(256, 1404002, 0.3), dict(n=8, step=4))]:
        want, st = oracle.encode(img, pv)
        with env(FIC_COARSE=coarse):
            enc = fic.encode(img, fic.CodecParams(**pv))
        assert_same(enc.mappings, want, f"coarse={coarse} {pv}")
        assert enc.stats == st


@pytest.mark.parametrize("acc", ["1", "0"])
@pytest.mark.parametrize("coarse", ["0", "1"])
def test_f16_accumulator_output_neutral(oracle, coarse, acc):
    """The full level with an fp16 accumulator (scan modes 5/6, the default after sparse levels
    and for large pools) and with an fp32 one (modes 0/1), each forced on small images of every
    range size (n = 2, 4, 8), with and without the whole-tile vote: identical codes and
    residual bits.
    The binary 0/255 image drives the operand/partial-sum overflow guard (ranges with a tiny
    bar relative to their norm get no bar)."""
    rng = np.random.default_rng(1404)
    binary = (rng.random((64, 64)) > 0.5).astype(np.uint8) * 255
    binary[:32, :32] = 128  # flat block: zero-variance ranges next to maximal-contrast ones
    cases = [(oracle.noise_image(64, 9), dict(n=4, step=2)), (oracle.smooth_image(64, 5), dict(n=8, step=2)),
             (images.ct_slice(256, 1404002, 0.3), dict(n=8, step=4)), (binary, dict(n=4, step=2)),
             (binary, dict(n=8, step=2)), (oracle.noise_image(64, 10), dict(n=2, step=1)),
             (oracle.smooth_image(64, 6), dict(n=2, step=3)), (binary, dict(n=2, step=1)),
             (images.ct_slice(128, 1404003, 0.5), dict(n=2, step=1))]
    for img, pv in cases:
        want, st = oracle.encode(img, pv)
        with env(FIC_F16ACC=acc, FIC_COARSE=coarse):
            enc = fic.encode(img, fic.CodecParams(**pv))
        assert_same(enc.mappings, want, f"f16acc={acc} coarse={coarse} {pv}")
        assert enc.stats == st


_SELECT_WANT = {}


@pytest.mark.parametrize("select", ["1", "2", "3"])
def test_sparse_selection_modes_output_neutral(oracle, select):
    """Every sparse-level selection (1 hit-first, 2 all-packed, 3 per-lane best: scan modes 2, 3,
    4) forced: a sparse level only lowers the bar, so codes and residual bits stay the
    reference's.  (The 256² n=4 step-2 pool, 123 tiles, is the one with a sparse level.)"""
    cases = [(oracle.noise_image(64, 9), dict(n=4, step=2)), (oracle.smooth_image(64, 5), dict(n=8, step=2)),
             (images.ct_slice(256, 1404002, 0.3), dict(n=8, step=4)),
             (images.ct_slice(256, 1404003, 0.3), dict(n=4, step=2))]
    for i, (img, pv) in enumerate(cases):
        if i not in _SELECT_WANT:
            _SELECT_WANT[i] = oracle.encode(img, pv)
        want, st = _SELECT_WANT[i]
        with env(FIC_SELECT=select):
            enc = fic.encode(img, fic.CodecParams(**pv))
        assert_same(enc.mappings, want, f"select={select} {pv}")
        assert enc.stats == st


@pytest.mark.parametrize("fused", ["0", "1"])
def test_fused_and_separate_evaluation(oracle, fused):
    """Survivors evaluated inside the scan kernel (default: consumer warps fed by the epilogue's
    chunks) or by the separate expand / eval / residual / winner kernels (FIC_FUSED=0): both give
    the reference's records, including with a survivor list small enough to overflow (the full
    level re-runs) and with every candidate surviving (exhaustive)."""
    cases = [(oracle.noise_image(64, 9), dict(n=4, step=2)), (oracle.smooth_image(64, 5), dict(n=8, step=2)),
             (images.ct_slice(256, 1404002, 0.3), dict(n=8, step=4)), (oracle.noise_image(64, 11), dict(n=2, step=1))]
    for img, pv in cases:
        want, st = oracle.encode(img, pv)
        for extra in (dict(), dict(FIC_LIST_CAP=3000), dict(FIC_DEBUG=1), dict(FIC_SEED=1), dict(FIC_EVAL_SPLIT=1),
                      dict(FIC_SPARSE_EXACT=1)):
            with env(FIC_FUSED=fused, **extra):
                enc = fic.encode(img, fic.CodecParams(**pv))
            assert_same(enc.mappings, want, f"fused={fused} {extra} {pv}")
            assert enc.stats == st


def test_random_parameter_sweep(oracle):
    """Seeded random sweep over the parameter space the reference accepts (range size, domain
    step, quantiser widths, s_max, shadow_eps) and image kinds (noise, smooth, binary, piecewise
    flat, the CT phantom) against the oracle: codes, residual bits and stats, through the
    default path (levels, selection, bars chosen per geometry)."""
    rng = np.random.default_rng(14040774)
    for trial in range(120):
        n = int(rng.choice([2, 4, 8]))
        side = int(rng.choice([s for s in (16, 32, 64, 128) if s >= 2 * n]))
        step = int(rng.integers(1, 2 * n + 1))
        pv = dict(n=n, step=step, s_bits=int(rng.integers(2, 9)), o_bits=int(rng.integers(3, 10)),
                  s_max=float(rng.choice([0.5, 0.75, 1.0, 1.5])),
                  shadow_eps=float(rng.choice([0.0, 0.0, 10.0, 300.0])))
        kind = trial % 5
        if kind == 0:
            img = oracle.noise_image(side, 1000 + trial)
        elif kind == 1:
            img = oracle.smooth_image(side, 1000 + trial)
        elif kind == 2:
            img = (rng.random((side, side)) > 0.5).astype(np.uint8) * 255
        elif kind == 3:
            img = oracle.smooth_image(side, 1000 + trial)
            img[: side // 2, : side // 3] = int(rng.integers(0, 256))
        else:
            img = images.ct_slice(side, 1404002 + trial, 0.2)
        want, st = oracle.encode(img, pv)
        enc = fic.encode(img, fic.CodecParams(**pv))
        assert_same(enc.mappings, want, f"trial {trial} {pv} kind {kind}")
        assert enc.stats == st, (trial, pv)


@pytest.mark.gpu
def test_encode_into_caller_buffers(oracle):
    """fic.encode(out=...): page-locked image and records (DMA both ways, the records copy
    riding in the replayed graph and retargeted to each call's buffer) and pageable ones give
    the same records as the plain call; a wrong buffer is refused."""
    import torch

    from paper_1404_0774_b200.abi import MAPPING_DTYPE

    img = images.ct_slice(256, 1404011, 0.4)
    p = fic.CodecParams(n=8, step=4)
    want, st = oracle.encode(img, dict(n=8, step=4))
    R = (256 // 8) ** 2
    pin_img = torch.empty(img.shape, dtype=torch.uint8, pin_memory=True).numpy()
    pin_img[:] = img
    outs = [torch.empty(R * 32, dtype=torch.uint8, pin_memory=True).numpy().view(MAPPING_DTYPE) for _ in range(2)]
    outs.append(np.zeros(R, MAPPING_DTYPE))
    for rep in range(3):  # eager, captured, replayed: each call into another buffer
        for k, o in enumerate(outs):
            o[:] = np.zeros(1, MAPPING_DTYPE)
            enc = fic.encode(pin_img if k != 2 else img, p, out=o)
            assert enc.mappings.base is o or np.shares_memory(enc.mappings, o)
            assert_same(o, want, f"out buffer {k} pass {rep}")
            assert enc.stats == st
    with pytest.raises(ValueError):
        fic.encode(img, p, out=np.zeros(R - 1, MAPPING_DTYPE))


@pytest.mark.gpu
@pytest.mark.parametrize("acc", ["1", "0"])
def test_near_threshold_candidates(oracle, acc):
    """Periodic textures with faint noise: whole families of domains are copies of each other
    up to a few grey levels, so each range has many candidates whose residuals tie or nearly tie
    with the bar, i.e. correlations that sit right at the scan's pruning threshold (and
    lexicographic ties the winner key must break by domain index).  Both accumulators, both
    sparse selections: identical codes and residual bits."""
    rng = np.random.default_rng(140401)
    cases = []
    for period, n, step, amp in [(8, 4, 2, 1), (16, 8, 4, 2), (4, 4, 1, 1), (12, 4, 3, 3), (8, 8, 2, 0)]:
        base = rng.integers(0, 256, (period, period))
        img = np.tile(base, (128 // period + 1, 128 // period + 1))[:128, :128]
        img = np.clip(img + rng.integers(-amp, amp + 1, img.shape), 0, 255).astype(np.uint8)
        cases.append((img, dict(n=n, step=step)))
    for img, pv in cases:
        want, st = oracle.encode(img, pv)
        for sel in ("0", "1"):
            with env(FIC_F16ACC=acc, FIC_F16SEL=sel):
                enc = fic.encode(img, fic.CodecParams(**pv))
            assert_same(enc.mappings, want, f"near-threshold acc={acc} sel={sel} {pv}")
            assert enc.stats == st


@pytest.mark.gpu
def test_batch_pipelined_caller_buffers(oracle):
    """encode_batch over several passes (FIC_BATCH_CHUNK=2: 5 slices = 3 pipelined passes),
    with page-locked volume and record buffers and with pageable ones: the same records as
    per-slice encodes, equal to the oracle on sampled slices."""
    import torch

    from paper_1404_0774_b200.abi import MAPPING_DTYPE

    vol = np.stack([images.ct_slice(128, 1404100 + i, 0.3) for i in range(5)])
    p = fic.CodecParams(n=8, step=4)
    per = (128 // 8) ** 2
    want = [fic.encode(s, p).mappings for s in vol]
    pin_vol = torch.empty(vol.shape, dtype=torch.uint8, pin_memory=True).numpy()
    pin_vol[:] = vol
    pin_out = torch.empty(5 * per * 32, dtype=torch.uint8, pin_memory=True).numpy().view(MAPPING_DTYPE)
    with env(FIC_BATCH_CHUNK=2):
        for src, out in ((vol, None), (pin_vol, pin_out), (pin_vol, None), (vol, pin_out)):
            encs, st = fic.encode_batch(src, p, out=out)
            for i, e in enumerate(encs):
                assert_same(e.mappings, want[i], f"slice {i}")
    for i in (0, 4):
        w, _ = oracle.encode(vol[i], dict(n=8, step=4))
        assert_same(want[i], w, f"oracle slice {i}")
