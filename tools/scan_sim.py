"""Simulates the dynamic pruning bar of a tiled scan (isometries on M, 128-domain tiles):
per tile, candidates with R* <= bar (bar = best exact R found so far, lagging `lag` tiles)
are "evaluated".  Counts evaluations per range for seed / prepass strategies.  CPU analysis only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.survivor_analysis import sym_src, quant, dequant  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402


def run(cfg, sample=None, tile=128, lag=1, prepass=0, seed9=True, chunks=1):
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    q, sq, sqq, flat = Oracle().domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
    PY = (W - 2 * n) // step + 1
    perm = np.array([[sym_src(s, i // n, i % n, n - 1)[0] * n + sym_src(s, i // n, i % n, n - 1)[1]
                      for i in range(N)] for s in range(8)])
    Qm = q[:, perm].astype(np.float64).reshape(D * 8, N)
    den = (N * sqq - sq * sq).astype(np.float64)
    RX = W // n
    R = RX * RX
    ridx = np.arange(R) if sample is None else np.linspace(0, R - 1, sample).astype(int)
    xs = (ridx % RX) * n
    ys = (ridx // RX) * n
    B = np.stack([img[y:y + n, x:x + n].reshape(-1) for x, y in zip(xs, ys)]).astype(np.float64)
    Sb = B.sum(1)
    Sbb = (B * B).sum(1)
    var = N * Sbb - Sb * Sb
    ssb = var / N
    ok = ~np.repeat(flat, 8)
    dd = np.where(ok, np.repeat(den, 8), 1.0)
    sqr = np.repeat(sq.astype(np.float64), 8)
    Sa, Saa = sqr * 0.25, np.repeat(sqq.astype(np.float64), 8) / 16
    tot_eval = 0
    tot_seed = 0
    per = []
    ch = 64
    ntile = (D + tile - 1) // tile
    for i0 in range(0, len(ridx), ch):
        b = B[i0:i0 + ch]
        sb = Sb[i0:i0 + ch, None]
        acc = b @ Qm.T
        num = N * acc - sqr[None, :] * sb
        rs = ssb[i0:i0 + ch, None] - num * num / (N * dd)[None, :]
        s = np.clip(4.0 * num / dd[None, :], -1.0, 1.0)
        sd = dequant(quant(s, 1.0, 5), 1.0, 5)
        o = np.clip((sb - s * Sa[None, :]) / N, -255, 255)
        od = dequant(quant(o, 255.0, 7), 255.0, 7)
        Rq = sd * sd * Saa + 2 * sd * od * Sa + N * od * od - 2 * sd * acc * 0.25 - 2 * od * sb + Sbb[i0:i0 + ch, None]
        rs[:, ~ok] = np.inf
        Rq[:, ~ok] = np.inf
        rs = rs.reshape(len(b), D, 8)
        Rq = Rq.reshape(len(b), D, 8)
        bar = np.full(len(b), np.inf)
        ev = np.zeros(len(b))
        if seed9:
            xi0 = np.clip((xs[i0:i0 + ch] - n // 2) // step, 0, None)
            yi0 = np.clip((ys[i0:i0 + ch] - n // 2) // step, 0, None)
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    xi, yi = xi0 + dx, yi0 + dy
                    okk = (xi >= 0) & (yi >= 0) & (xi < PY) & (yi < PY)
                    d = np.where(okk, xi * PY + yi, 0)
                    v = Rq[np.arange(len(b)), d].min(1)
                    bar = np.minimum(bar, np.where(okk, v, np.inf))
            tot_seed += 72 * len(b)
        if prepass:
            # sparse pass over every `prepass`-th tile with the seed bar (lag ignored)
            for t in range(0, ntile, prepass):
                blk = slice(t * tile, min(D, (t + 1) * tile))
                surv = rs[:, blk] <= bar[:, None, None] * (1 + 1e-3)
                ev += surv.sum((1, 2))
                bar = np.minimum(bar, np.where(surv, Rq[:, blk], np.inf).min((1, 2)))
        # full scan, chunked: each chunk starts from the same (post-prepass) bar and runs in parallel
        cb = bar.copy()
        bounds = np.linspace(0, ntile, chunks + 1).astype(int)
        pend = []
        for c in range(chunks):
            bar_c = cb.copy()
            hist = []
            for t in range(bounds[c], bounds[c + 1]):
                blk = slice(t * tile, min(D, (t + 1) * tile))
                surv = rs[:, blk] <= bar_c[:, None, None] * (1 + 1e-3)
                ev += surv.sum((1, 2))
                hist.append(np.where(surv, Rq[:, blk], np.inf).min((1, 2)))
                if len(hist) > lag:
                    bar_c = np.minimum(bar_c, hist[-1 - lag])
        act = var[i0:i0 + ch] > 0
        per.append(ev[act])
        tot_eval += ev[act].sum()
    per = np.concatenate(per)
    print(f"{cfg} tile={tile} lag={lag} prepass={prepass} seed9={seed9} chunks={chunks}: evaluations/range mean "
          f"{per.mean():.1f} p50 {np.median(per):.0f} p99 {np.quantile(per, .99):.0f} max {per.max():.0f}")


def static_levels(cfg, sample=None, tile=128, schemes=((64, 8), (32,), (256, 16), (128, 8), (16,)), seed_h=1):
    """Static multi-level scheme: seed (9 local domains) -> level strides (sparse tile subsets,
    each scanned against the bar of the previous levels, all survivors evaluated) -> full scan."""
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    q, sq, sqq, flat = Oracle().domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
    PY = (W - 2 * n) // step + 1
    perm = np.array([[sym_src(s, i // n, i % n, n - 1)[0] * n + sym_src(s, i // n, i % n, n - 1)[1]
                      for i in range(N)] for s in range(8)])
    Qm = q[:, perm].astype(np.float64).reshape(D * 8, N)
    den = (N * sqq - sq * sq).astype(np.float64)
    RX = W // n
    R = RX * RX
    ridx = np.arange(R) if sample is None else np.linspace(0, R - 1, sample).astype(int)
    xs = (ridx % RX) * n
    ys = (ridx // RX) * n
    B = np.stack([img[y:y + n, x:x + n].reshape(-1) for x, y in zip(xs, ys)]).astype(np.float64)
    Sb = B.sum(1)
    Sbb = (B * B).sum(1)
    var = N * Sbb - Sb * Sb
    ssb = var / N
    ok = ~np.repeat(flat, 8)
    dd = np.where(ok, np.repeat(den, 8), 1.0)
    sqr = np.repeat(sq.astype(np.float64), 8)
    Sa, Saa = sqr * 0.25, np.repeat(sqq.astype(np.float64), 8) / 16
    ntile = (D + tile - 1) // tile
    res = {sc: [] for sc in schemes}
    ch = int(os.environ.get("CH", "64"))
    for i0 in range(0, len(ridx), ch):
        b = B[i0:i0 + ch]
        sb = Sb[i0:i0 + ch, None]
        acc = b @ Qm.T
        num = N * acc - sqr[None, :] * sb
        rs = ssb[i0:i0 + ch, None] - num * num / (N * dd)[None, :]
        s = np.clip(4.0 * num / dd[None, :], -1.0, 1.0)
        sd = dequant(quant(s, 1.0, 5), 1.0, 5)
        o = np.clip((sb - s * Sa[None, :]) / N, -255, 255)
        od = dequant(quant(o, 255.0, 7), 255.0, 7)
        Rq = sd * sd * Saa + 2 * sd * od * Sa + N * od * od - 2 * sd * acc * 0.25 - 2 * od * sb + Sbb[i0:i0 + ch, None]
        rs[:, ~ok] = np.inf
        Rq[:, ~ok] = np.inf
        rs = rs.reshape(len(b), D, 8)
        Rq = Rq.reshape(len(b), D, 8)
        act = var[i0:i0 + ch] > 0
        seed = np.full(len(b), np.inf)
        xi0 = np.clip((xs[i0:i0 + ch] - n // 2) // step, 0, None)
        yi0 = np.clip((ys[i0:i0 + ch] - n // 2) // step, 0, None)
        for dx in range(-seed_h, seed_h + 1):
            for dy in range(-seed_h, seed_h + 1):
                xi, yi = xi0 + dx, yi0 + dy
                okk = (xi >= 0) & (yi >= 0) & (xi < PY) & (yi < PY)
                d = np.where(okk, xi * PY + yi, 0)
                v = Rq[np.arange(len(b)), d].min(1)
                seed = np.minimum(seed, np.where(okk, v, np.inf))
        for sc in schemes:
            bar = seed.copy()
            counts = []
            for stride in list(sc) + [1]:
                tiles = np.zeros(D, bool)
                for t in range(0, ntile, stride):
                    tiles[t * tile:(t + 1) * tile] = True
                surv = rs[:, tiles] <= bar[:, None, None] * (1 + 1e-3)
                counts.append(surv.sum((1, 2)))
                bar = np.minimum(bar, np.where(surv, Rq[:, tiles], np.inf).min((1, 2)))
            res[sc].append(np.stack(counts, 1)[act])
    for sc, v in res.items():
        v = np.concatenate(v)
        print(f"{cfg} levels {sc}+full: survivors/range per level mean {np.round(v.mean(0), 1)} "
              f"total {v.sum(1).mean():.1f}  p99 total {np.quantile(v.sum(1), .99):.0f}  max level {v.max(0)}")


if __name__ == "__main__":
    cfg = sys.argv[1]
    sample = int(sys.argv[2]) if len(sys.argv) > 2 else None
    if "--static" in sys.argv:
        static_levels(cfg, sample)
        sys.exit(0)
    for kw in [dict(), dict(lag=4), dict(prepass=16), dict(prepass=16, lag=4), dict(prepass=16, chunks=4, lag=4),
               dict(seed9=False, lag=4)]:
        run(cfg, sample, **kw)


def dynamic_bitrev(cfg, sample=None, tile=128, lags=(1, 4, 16), seed_h=1):
    """Single pass over tiles in bit-reversed order, bar = best exact R of the survivors
    evaluated so far (visible `lag` tiles later)."""
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    q, sq, sqq, flat = Oracle().domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
    PY = (W - 2 * n) // step + 1
    perm = np.array([[sym_src(s, i // n, i % n, n - 1)[0] * n + sym_src(s, i // n, i % n, n - 1)[1]
                      for i in range(N)] for s in range(8)])
    Qm = q[:, perm].astype(np.float64).reshape(D * 8, N)
    den = (N * sqq - sq * sq).astype(np.float64)
    RX = W // n
    R = RX * RX
    ridx = np.arange(R) if sample is None else np.linspace(0, R - 1, sample).astype(int)
    xs = (ridx % RX) * n
    ys = (ridx // RX) * n
    B = np.stack([img[y:y + n, x:x + n].reshape(-1) for x, y in zip(xs, ys)]).astype(np.float64)
    Sb = B.sum(1)
    Sbb = (B * B).sum(1)
    var = N * Sbb - Sb * Sb
    ssb = var / N
    ok = ~np.repeat(flat, 8)
    dd = np.where(ok, np.repeat(den, 8), 1.0)
    sqr = np.repeat(sq.astype(np.float64), 8)
    Sa, Saa = sqr * 0.25, np.repeat(sqq.astype(np.float64), 8) / 16
    ntile = (D + tile - 1) // tile
    bits = int(np.ceil(np.log2(max(ntile, 2))))
    order = sorted(range(ntile), key=lambda t: int(format(t, f'0{bits}b')[::-1], 2))
    res = {lag: [] for lag in lags}
    ch = int(os.environ.get("CH", "64"))
    for i0 in range(0, len(ridx), ch):
        b = B[i0:i0 + ch]
        sb = Sb[i0:i0 + ch, None]
        acc = b @ Qm.T
        num = N * acc - sqr[None, :] * sb
        rs = ssb[i0:i0 + ch, None] - num * num / (N * dd)[None, :]
        s = np.clip(4.0 * num / dd[None, :], -1.0, 1.0)
        sd = dequant(quant(s, 1.0, 5), 1.0, 5)
        o = np.clip((sb - s * Sa[None, :]) / N, -255, 255)
        od = dequant(quant(o, 255.0, 7), 255.0, 7)
        Rq = sd * sd * Saa + 2 * sd * od * Sa + N * od * od - 2 * sd * acc * 0.25 - 2 * od * sb + Sbb[i0:i0 + ch, None]
        rs[:, ~ok] = np.inf
        Rq[:, ~ok] = np.inf
        rs = rs.reshape(len(b), D, 8)
        Rq = Rq.reshape(len(b), D, 8)
        act = var[i0:i0 + ch] > 0
        seed = np.full(len(b), np.inf)
        xi0 = np.clip((xs[i0:i0 + ch] - n // 2) // step, 0, None)
        yi0 = np.clip((ys[i0:i0 + ch] - n // 2) // step, 0, None)
        for dx in range(-seed_h, seed_h + 1):
            for dy in range(-seed_h, seed_h + 1):
                xi, yi = xi0 + dx, yi0 + dy
                okk = (xi >= 0) & (yi >= 0) & (xi < PY) & (yi < PY)
                d = np.where(okk, xi * PY + yi, 0)
                v = Rq[np.arange(len(b)), d].min(1)
                seed = np.minimum(seed, np.where(okk, v, np.inf))
        for lag in lags:
            bar = seed.copy()
            hist = []
            cnt = np.zeros(len(b))
            for t in order:
                blk = slice(t * tile, min(D, (t + 1) * tile))
                surv = rs[:, blk] <= bar[:, None, None] * (1 + 1e-3)
                cnt += surv.sum((1, 2))
                hist.append(np.where(surv, Rq[:, blk], np.inf).min((1, 2)))
                if len(hist) > lag:
                    bar = np.minimum(bar, hist[-1 - lag])
            res[lag].append(cnt[act])
    for lag, v in res.items():
        v = np.concatenate(v)
        print(f"{cfg} bit-reversed single pass, lag {lag}: survivors/range mean {v.mean():.1f} p99 {np.quantile(v, .99):.0f}")
