"""Deterministic synthetic grayscale inputs for the benchmark configurations.

The reference ships no phantom / CT / X-ray generators, so these are
defined here, seeded from std::mt19937 raw draws (numpy's MT19937 with legacy seeding
reproduces them bit for bit; proj/tests/testimg.hpp:11-12 pins the engine, not a
distribution).  All images are uint8, square, power-of-two sides.

    phantom(256, 1404001)          cfg1: Shepp-Logan-style ellipse sum + uniform +-2 noise
    ct_slice(512, 1404002)         cfg2/cfg3: elliptical body, bone rim, organs, noise sigma~4
    xray(2048, 1404004)            cfg4: smooth attenuation gradient + rib-like bands + noise
    volume(512, 512, 1404005)      cfg5: CT slices whose radii vary with z (seed 1404005+z)
    noise_image / smooth_image     the reference's own fixtures (testimg.hpp:13-59)
"""
import numpy as np


class _Raw:
    """std::mt19937(seed) raw 32-bit draws."""

    def __init__(self, seed):
        self.bg = np.random.MT19937()
        self.bg._legacy_seeding(int(seed) & 0xFFFFFFFF)

    def u32(self, n):
        return self.bg.random_raw(int(n)).astype(np.uint64)

    def unit(self, n=1):
        return self.u32(n).astype(np.float64) / 4294967296.0


def noise_image(side, seed):
    """testimg.hpp:13-21: uniform noise, one raw draw per pixel (row-major)."""
    r = _Raw(seed)
    return (r.u32(side * side) & 0xFF).astype(np.uint8).reshape(side, side)


def smooth_image(side, seed):
    """testimg.hpp:26-59: ramp plus four cosine bumps (uses libm cos via numpy)."""
    r = _Raw(seed)
    bumps = []
    for _ in range(4):
        u = r.unit(4)
        bumps.append((1.0 + u[0] * 3.0, 1.0 + u[1] * 3.0, u[2] * 6.283185307179586, 20.0 + u[3] * 25.0))
    g = r.unit(2)
    gx, gy = g[0] * 60.0 - 30.0, g[1] * 60.0 - 30.0
    y, x = np.mgrid[0:side, 0:side].astype(np.float64)
    u, v = x / side, y / side
    z = 128.0 + gx * (u - 0.5) + gy * (v - 0.5)
    for fx, fy, ph, amp in bumps:
        z = z + amp * np.cos(6.283185307179586 * (fx * u + fy * v) + ph)
    return _lround_nonneg(np.clip(z, 0.0, 255.0)).astype(np.uint8)


def _lround_nonneg(x):
    """std::lround for x >= 0 (half away from zero), exact: x - trunc(x) has no rounding."""
    t = np.trunc(x)
    return t + ((x - t) >= 0.5)


def _noise_sigma(r, shape, sigma):
    """Approximately Gaussian noise: sum of 12 uniforms minus 6 (Irwin-Hall)."""
    u = r.unit(int(np.prod(shape)) * 12).reshape(-1, 12).sum(axis=1) - 6.0
    return (u * sigma).reshape(shape)


def _ellipse(X, Y, cx, cy, ax, ay, theta):
    c, s = np.cos(theta), np.sin(theta)
    xr = (X - cx) * c + (Y - cy) * s
    yr = -(X - cx) * s + (Y - cy) * c
    return (xr / ax) ** 2 + (yr / ay) ** 2 <= 1.0


# Modified Shepp-Logan: (intensity, a, b, x0, y0, phi degrees)
_SHEPP = [
    (1.0, 0.69, 0.92, 0.0, 0.0, 0),
    (-0.8, 0.6624, 0.874, 0.0, -0.0184, 0),
    (-0.2, 0.11, 0.31, 0.22, 0.0, -18),
    (-0.2, 0.16, 0.41, -0.22, 0.0, 18),
    (0.1, 0.21, 0.25, 0.0, 0.35, 0),
    (0.1, 0.046, 0.046, 0.0, 0.1, 0),
    (0.1, 0.046, 0.046, 0.0, -0.1, 0),
    (0.1, 0.046, 0.023, -0.08, -0.605, 0),
    (0.1, 0.023, 0.023, 0.0, -0.606, 0),
    (0.1, 0.023, 0.046, 0.06, -0.605, 0),
]


def phantom(side=256, seed=1404001):
    """cfg1: Shepp-Logan-style ellipse sum scaled to [0, 255] plus uniform integer noise in [-2, 2]."""
    r = _Raw(seed)
    c = (np.arange(side, dtype=np.float64) + 0.5) / side * 2.0 - 1.0
    X, Y = np.meshgrid(c, -c)
    img = np.zeros((side, side))
    for inten, a, b, x0, y0, phi in _SHEPP:
        img += inten * _ellipse(X, Y, x0, y0, a, b, np.deg2rad(phi))
    img = (img - img.min()) / (img.max() - img.min()) * 235.0 + 10.0
    noise = (r.u32(side * side) % 5).astype(np.float64).reshape(side, side) - 2.0
    return np.clip(np.rint(img + noise), 0, 255).astype(np.uint8)


def ct_slice(side=512, seed=1404002, z=0.0):
    """cfg2/cfg3: elliptical body (soft tissue ~100, bone rim ~220, air 0), a few organs
    drawn from the seed, Gaussian-like noise sigma ~4 (air included)."""
    r = _Raw(seed)
    c = (np.arange(side, dtype=np.float64) + 0.5) / side * 2.0 - 1.0
    X, Y = np.meshgrid(c, c)
    wobble = 1.0 + 0.08 * np.sin(2.0 * np.pi * z)
    ax, ay = 0.82 * wobble, 0.62 / wobble
    img = np.zeros((side, side))
    body = _ellipse(X, Y, 0.0, 0.0, ax, ay, 0.0)
    img[body] = 100.0
    rim = body & ~_ellipse(X, Y, 0.0, 0.0, ax - 0.05, ay - 0.05, 0.0)
    img[rim] = 220.0
    u = r.unit(6 * 8).reshape(8, 6)
    for k in range(8):
        cx, cy = (u[k, 0] - 0.5) * ax, (u[k, 1] - 0.5) * ay
        a_, b_ = 0.05 + 0.15 * u[k, 2], 0.05 + 0.12 * u[k, 3]
        inten = 40.0 + 110.0 * u[k, 4]
        img[_ellipse(X, Y, cx, cy, a_, b_, np.pi * u[k, 5]) & body & ~rim] = inten
    spine = _ellipse(X, Y, 0.0, ay * 0.6, 0.08, 0.07, 0.0)
    img[spine] = 230.0
    img += _noise_sigma(r, img.shape, 4.0)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def xray(side=2048, seed=1404004):
    """cfg4: smooth attenuation gradient + rib-like cosine bands + lung fields + noise."""
    r = _Raw(seed)
    c = (np.arange(side, dtype=np.float64) + 0.5) / side
    X, Y = np.meshgrid(c, c)
    u = r.unit(6)
    base = 60.0 + 90.0 * np.exp(-((X - 0.5) ** 2) / (0.18 + 0.05 * u[0])) * (0.7 + 0.3 * Y)
    ribs = 25.0 * np.maximum(0.0, np.cos(2.0 * np.pi * (9.0 + 2.0 * u[1]) * (Y + 0.15 * (X - 0.5) ** 2))) ** 3
    lungs = (_ellipse(X, Y, 0.32, 0.48, 0.14, 0.3, 0.05) | _ellipse(X, Y, 0.68, 0.48, 0.14, 0.3, -0.05))
    img = base + ribs * lungs - 35.0 * lungs + 40.0 * _ellipse(X, Y, 0.5, 0.55, 0.045, 0.42, 0.0)
    img += _noise_sigma(r, img.shape, 3.0)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def volume(count=512, side=512, seed=1404005):
    """cfg5: `count` CT slices; slice z uses seed 1404005+z and radii varying with z."""
    return np.stack([ct_slice(side, seed + z, z / max(count, 1)) for z in range(count)])


def volume_slices(first, count, total=512, side=512, seed=1404005):
    """Slices [first, first + count) of volume(total, side, seed) (a rank's shard of cfg5)."""
    z = range(first, min(total, first + count))
    return np.stack([ct_slice(side, seed + k, k / max(total, 1)) for k in z])


CONFIGS = {
    # name: (generator, n, step)
    "cfg1": (lambda: phantom(256, 1404001), 8, 8),
    "cfg2": (lambda: ct_slice(512, 1404002), 8, 4),
    "cfg3": (lambda: ct_slice(512, 1404002), 4, 2),
    "cfg4": (lambda: xray(2048, 1404004), 8, 2),
}
