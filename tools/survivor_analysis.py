"""Offline (CPU, numpy) analysis of the pruning bound: how many candidates survive the
unconstrained least-squares bound R* <= bar for various bars.  Used to choose the GPU
matcher's seeding strategy; not part of the product."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle, Reference  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402


def sym_src(s, r, c, m):
    return [(r, c), (m - c, r), (m - r, m - c), (c, m - r), (r, m - c), (m - r, c), (c, r), (m - c, m - r)][s]


def main(cfg="cfg2", sample=None, workers=8):
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    O = Oracle()
    q, sq, sqq, flat = O.domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
    perm = np.array([[sym_src(s, i // n, i % n, n - 1)[0] * n + sym_src(s, i // n, i % n, n - 1)[1]
                      for i in range(N)] for s in range(8)])
    Q8 = q[:, perm].astype(np.float64)  # D x 8 x N : element (d, s, i) = q[d, perm_s(i)]
    den = N * sqq - sq * sq
    RX = W // n
    R = RX * RX
    ridx = np.arange(R) if sample is None else np.linspace(0, R - 1, sample).astype(int)
    xs = (ridx % RX) * n
    ys = (ridx // RX) * n
    B = np.stack([img[y:y + n, x:x + n].reshape(-1) for x, y in zip(xs, ys)]).astype(np.float64)
    Sb = B.sum(1)
    var = N * (B * B).sum(1) - Sb * Sb
    ssb = var / N
    t = time.time()
    ref = Reference()
    if sample is None:
        recs, st = ref.encode(img, dict(n=n, step=step), workers=workers)
    else:
        recs = np.array([ref.encode_range(img, int(x), int(y), dict(n=n, step=step))[0] for x, y in zip(xs, ys)])
    best = recs["residual"].astype(np.float64)
    print(f"{cfg}: R={R} sampled={len(ridx)} D={D} flat={flat.sum()} ref {time.time() - t:.1f}s")
    Qm = Q8.reshape(D * 8, N)
    ok = ~np.repeat(flat, 8)
    dd = np.repeat(den.astype(np.float64), 8)
    sqr = np.repeat(sq.astype(np.float64), 8)
    counts = {k: 0 for k in ["le_best", "le_best_1.1", "le_best_1.5", "le_best_2", "total"]}
    rstar_min = np.empty(len(ridx))
    ch = 256
    for i0 in range(0, len(ridx), ch):
        b = B[i0:i0 + ch]
        acc = b @ Qm.T
        num = N * acc - sqr[None, :] * Sb[i0:i0 + ch, None]
        rs = ssb[i0:i0 + ch, None] - num * num / (N * np.where(ok, dd, 1.0))[None, :]
        rs[:, ~ok] = np.inf
        act = var[i0:i0 + ch] > 0
        rs[~act] = np.inf
        bb = best[i0:i0 + ch, None]
        counts["le_best"] += int((rs <= bb).sum())
        counts["le_best_1.1"] += int((rs <= bb * 1.1 + 1e-9).sum())
        counts["le_best_1.5"] += int((rs <= bb * 1.5 + 1e-9).sum())
        counts["le_best_2"] += int((rs <= bb * 2 + 1e-9).sum())
        counts["total"] += int(act.sum()) * int(ok.sum())
        rstar_min[i0:i0 + ch] = rs.min(1)
    tot = counts["total"]
    for k, v in counts.items():
        print(f"  {k:12s} {v:12d}  {v / tot * 100:8.4f}%  per range {v / len(ridx):9.1f}")
    act = var > 0
    ratio = best[act] / np.maximum(rstar_min[act], 1e-12)
    print("  best/minR* quantiles", np.quantile(ratio, [0.1, 0.5, 0.9, 0.99]))
    print("  best/ssb quantiles", np.quantile(best[act] / ssb[act], [0.1, 0.5, 0.9, 0.99]))


def quant(v, M, bits):
    mc = (1 << bits) - 1
    code = np.floor((v + M) / (2 * M) * mc + 0.5)
    code = np.clip(code, 1, mc)
    return np.where(v == 0.0, 0, code)


def dequant(c, M, bits):
    mc = (1 << bits) - 1
    return np.where(c == 0, 0.0, -M + 2 * M * (c / mc))


def strategies(cfg="cfg2", sample=None, ks=(1, 2, 4, 8, 16, 32, 64)):
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    O = Oracle()
    q, sq, sqq, flat = O.domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
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
    sqqr = np.repeat(sqq.astype(np.float64), 8)
    Sa, Saa = sqr * 0.25, sqqr / 16
    res = {k: [] for k in ks}
    full = []
    prepass = {32: [], 512: []}
    ch = int(os.environ.get("CH", "128"))
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
        Sab = acc * 0.25
        Rq = sd * sd * Saa + 2 * sd * od * Sa + N * od * od - 2 * sd * Sab - 2 * od * sb + Sbb[i0:i0 + ch, None]
        rs[:, ~ok] = np.inf
        Rq[:, ~ok] = np.inf
        act = var[i0:i0 + ch] > 0
        best = Rq.min(1)
        # group (domain) score = min over isometries of R*
        g = rs.reshape(len(b), D, 8).min(2)
        order = np.argsort(g, axis=1)
        Rqg = Rq.reshape(len(b), D, 8).min(2)
        for k in ks:
            topk = order[:, :k]
            bar = np.take_along_axis(Rqg, topk, 1).min(1)
            surv = (rs <= bar[:, None] * (1 + 1e-6)).sum(1)
            kth = np.take_along_axis(g, order[:, k - 1:k], 1)[:, 0]
            covered = kth > bar  # every candidate with R* <= bar is inside the top-k groups
            res[k].append(np.stack([surv[act], covered[act], (bar / best)[act]], 1))
        for stp in prepass:
            sel = np.zeros(D, bool)
            sel[::stp * 16] = True  # every stp-th 16-domain tile (first domain of it) ~ sparse
            tiles = np.zeros(D, bool)
            for t0 in range(0, D, 16 * stp):
                tiles[t0:t0 + 16] = True
            bar = Rqg[:, tiles].min(1)
            surv = (rs <= bar[:, None] * (1 + 1e-6)).sum(1)
            prepass[stp].append(np.stack([surv[act], (bar / best)[act]], 1))
        full.append(((rs <= best[:, None] * (1 + 1e-6)).sum(1))[act])
    full = np.concatenate(full)
    print(f"{cfg}: perfect-bar survivors/range mean {full.mean():.1f} p50 {np.median(full):.0f} p99 {np.quantile(full, .99):.0f}"
          f" max {full.max()}")
    for stp, v in prepass.items():
        v = np.concatenate(v)
        print(f"  prepass 1/{stp}: survivors/range mean {v[:, 0].mean():9.1f} p99 {np.quantile(v[:, 0], .99):9.0f} "
              f"bar/best p50 {np.median(v[:, 1]):.4f}")
    for k, v in res.items():
        v = np.concatenate(v)
        print(f"  top-{k:3d} by R*: survivors/range mean {v[:, 0].mean():9.1f} p99 {np.quantile(v[:, 0], .99):9.0f}"
              f"  covered {v[:, 1].mean() * 100:6.2f}%  bar==best {np.mean(v[:, 2] <= 1 + 1e-12) * 100:6.2f}%"
              f"  bar/best p90 {np.quantile(v[:, 2], .9):.4f}")


def quant_filter(cfg="cfg2", p=None):
    """Survivors of the unconstrained bound (R* <= best) against those of the exact quantised
    residual (s, o quantised as the reference does: R_q = parabola + N o_gap^2 <= best), and
    how many (range, 32-domain warp chunk) groups each leaves for the scan epilogue."""
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    O = Oracle()
    q, sq, sqq, flat = O.domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
    perm = np.array([[sym_src(s, i // n, i % n, n - 1)[0] * n + sym_src(s, i // n, i % n, n - 1)[1]
                      for i in range(N)] for s in range(8)])
    Qm = q[:, perm].astype(np.float64).reshape(D * 8, N)
    den = (N * sqq - sq * sq).astype(np.float64)
    recs, _ = O.encode(img, dict(n=n, step=step))
    best = recs["residual"].astype(np.float64)
    RX = W // n
    R = RX * RX
    xs = (np.arange(R) % RX) * n
    ys = (np.arange(R) // RX) * n
    B = np.stack([img[y:y + n, x:x + n].reshape(-1) for x, y in zip(xs, ys)]).astype(np.float64)
    Sb = B.sum(1)
    var = N * (B * B).sum(1) - Sb * Sb
    ssb = var / N
    ok = ~np.repeat(flat, 8)
    dd = np.where(ok, np.repeat(den, 8), 1.0)
    sqr = np.repeat(sq.astype(np.float64), 8)
    smax, sb_, ob_ = 1.0, 5, 7
    nrm = O.normalize(dict(n=n, step=step))
    smax, sb_, ob_ = nrm.s_max, nrm.s_bits, nrm.o_bits
    chunk = np.arange(D * 8) // 8 // 32  # the scan's 32-domain warp chunks
    tot = dict(rstar=0, rq=0, g_rstar=0, g_rq=0)
    per_range = []
    for i0 in range(0, R, 64):
        b = B[i0:i0 + 64]
        acc = b @ Qm.T
        num = N * acc - sqr[None, :] * Sb[i0:i0 + 64, None]
        rs = ssb[i0:i0 + 64, None] - num * num / (N * dd)[None, :]
        act = (var[i0:i0 + 64] > 0)[:, None] & ok[None, :]
        bb = best[i0:i0 + 64, None]
        hit = act & (rs <= bb)
        sc = np.clip(4.0 * num / dd[None, :], -smax, smax)
        s_deq = dequant(quant(sc, smax, sb_), smax, sb_)
        cov = num * 0.25 / N
        var_a = dd[None, :] * 0.0625 / N
        par = ssb[i0:i0 + 64, None] - 2 * s_deq * cov + s_deq * s_deq * var_a
        sa = sqr[None, :] * 0.25
        o = np.clip((Sb[i0:i0 + 64, None] - sc * sa) / N, -255, 255)
        o_deq = dequant(quant(o, 255.0, ob_), 255.0, ob_)
        og = o_deq - (Sb[i0:i0 + 64, None] - s_deq * sa) / N
        rq = par + N * og * og
        hq = hit & (rq <= bb * (1 + 1e-6) + 1e-6)
        # bars after sparse levels over every k-th 128-domain tile (exact R_q minimum there)
        tile = (np.arange(D * 8) // 8) // 128
        for k in (64, 8, 4, 2):
            rqk = np.where(act & (tile % k == 0)[None, :], rq, np.inf).min(1, keepdims=True)
            tot.setdefault(f"bar{k}", 0)
            tot[f"bar{k}"] += int((act & (rs <= rqk)).sum())
            tot.setdefault(f"lvl{k}", 0)
            tot[f"lvl{k}"] += int((act & (rs <= rqk) & (tile % k == 0)[None, :]).sum())
        tot["rstar"] += int(hit.sum())
        tot["rq"] += int(hq.sum())
        for h, key in ((hit, "g_rstar"), (hq, "g_rq")):
            rr, cc = np.nonzero(h)
            tot[key] += len(np.unique(rr.astype(np.int64) * (1 << 20) + chunk[cc]))
        per_range.extend(hit.sum(1).tolist())
    pr = np.array(per_range)
    print(f"{cfg}: R={R} D={D}  R*-survivors {tot['rstar']} ({tot['rstar'] / R:.1f}/range) in {tot['g_rstar']} groups; "
          f"R_q-survivors {tot['rq']} ({tot['rq'] / R:.2f}/range) in {tot['g_rq']} groups")
    print("  full-level R*-survivors with the bar of a sparse level over every k-th tile:",
          {k: tot[f"bar{k}"] for k in (64, 8, 4, 2)}, " level-k own survivors:", {k: tot[f"lvl{k}"] for k in (64, 8, 4, 2)})
    print("  R*-survivors per range quantiles (50/90/99/max):", np.quantile(pr, [0.5, 0.9, 0.99]), pr.max())
    print("  ranges holding half of the survivors:", int(np.searchsorted(np.cumsum(np.sort(pr)[::-1]), pr.sum() / 2)))


def level_schemes(cfg="cfg2", schemes=None):
    """Survivors per scan level for level schemes, with the bar each level starts from (the
    3x3 local seed, then the exact minimum over every tile scanned so far).  A scheme is a list
    of tile strides; "rescan" levels scan every stride-k tile, "partition" levels skip tiles an
    earlier level scanned."""
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    W = img.shape[0]
    N = n * n
    O = Oracle()
    nrm = O.normalize(dict(n=n, step=step))
    q, sq, sqq, flat = O.domain_pool(img, dict(n=n, step=step))
    D = q.shape[0]
    PY = (W - 2 * n) // step + 1
    perm = np.array([[sym_src(s, i // n, i % n, n - 1)[0] * n + sym_src(s, i // n, i % n, n - 1)[1]
                      for i in range(N)] for s in range(8)])
    Qm = q[:, perm].astype(np.float64).reshape(D * 8, N)
    den = (N * sqq - sq * sq).astype(np.float64)
    RX = W // n
    R = RX * RX
    xs = (np.arange(R) % RX) * n
    ys = (np.arange(R) // RX) * n
    B = np.stack([img[y:y + n, x:x + n].reshape(-1) for x, y in zip(xs, ys)]).astype(np.float64)
    Sb = B.sum(1)
    var = N * (B * B).sum(1) - Sb * Sb
    ssb = var / N
    ok = ~np.repeat(flat, 8)
    dd = np.where(ok, np.repeat(den, 8), 1.0)
    sqr = np.repeat(sq.astype(np.float64), 8)
    tile = (np.arange(D * 8) // 8) // 128
    T = tile.max() + 1
    schemes = schemes or [("rescan", [64, 8, 1]), ("partition", [64, 8, 1]), ("partition", [64, 16, 4, 1]),
                          ("partition", [32, 8, 2, 1]), ("partition", [16, 4, 1]), ("partition", [64, 16, 4, 2, 1]),
                          ("partition", [128, 32, 8, 2, 1])]
    out = {i: [0] * len(sc[1]) for i, sc in enumerate(schemes)}
    tiles = {i: [] for i in range(len(schemes))}
    for i, (kind, lv) in enumerate(schemes):
        done = np.zeros(T, bool)
        for k in lv:
            sel = (np.arange(T) % k == 0) & (~done if kind == "partition" else True)
            tiles[i].append(int(sel.sum()))
            done |= sel
    for i0 in range(0, R, 64):
        sl = slice(i0, i0 + 64)
        acc = B[sl] @ Qm.T
        num = N * acc - sqr[None, :] * Sb[sl, None]
        rs = ssb[sl, None] - num * num / (N * dd)[None, :]
        act = (var[sl] > 0)[:, None] & ok[None, :]
        sc = np.clip(4.0 * num / dd[None, :], -nrm.s_max, nrm.s_max)
        s_deq = dequant(quant(sc, nrm.s_max, nrm.s_bits), nrm.s_max, nrm.s_bits)
        sa = sqr[None, :] * 0.25
        par = ssb[sl, None] - 2 * s_deq * num * 0.25 / N + s_deq * s_deq * dd[None, :] * 0.0625 / N
        o = np.clip((Sb[sl, None] - sc * sa) / N, -255, 255)
        og = dequant(quant(o, 255.0, nrm.o_bits), 255.0, nrm.o_bits) - (Sb[sl, None] - s_deq * sa) / N
        rq = np.where(act, par + N * og * og, np.inf)
        # seed bar: 3x3 domains around the range centre
        seed = np.full(rq.shape[0], np.inf)
        for r in range(rq.shape[0]):
            x0, y0 = xs[i0 + r], ys[i0 + r]
            xi0 = min(max((x0 - n // 2) // step, 0), PY - 1)
            yi0 = min(max((y0 - n // 2) // step, 0), PY - 1)
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    xi, yi = xi0 + dx, yi0 + dy
                    if 0 <= xi < PY and 0 <= yi < PY:
                        d = xi * PY + yi
                        seed[r] = min(seed[r], rq[r, d * 8:(d + 1) * 8].min())
        for i, (kind, lv) in enumerate(schemes):
            bar = seed.copy()
            done = np.zeros(T, bool)
            for li, k in enumerate(lv):
                sel_t = (np.arange(T) % k == 0) & (~done if kind == "partition" else True)
                sel = sel_t[tile]
                out[i][li] += int((act & sel[None, :] & (rs <= bar[:, None])).sum())
                bar = np.minimum(bar, np.where(sel[None, :], rq, np.inf).min(1))
                done |= sel_t
    for i, (kind, lv) in enumerate(schemes):
        print(f"  {kind:9s} {str(lv):22s} tiles {tiles[i]} (sum {sum(tiles[i])} of {T})  survivors {out[i]} "
              f"sum {sum(out[i])}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "levels":
        level_schemes(*(sys.argv[2:3] or ["cfg2"]))
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "quant":
        quant_filter(*(sys.argv[2:3] or ["cfg2"]))
        sys.exit(0)
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    sample = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else None
    (strategies if "--strat" in sys.argv else main)(cfg, sample)
