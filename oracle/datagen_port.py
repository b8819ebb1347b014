"""TEST INFRASTRUCTURE: numpy port of the on-device BASELINE generator
(paper_2406_10262_b200/csrc/nsw_datagen.cu), used only to check the device
generator on user slices.  Philox4x32-10 in uint64 numpy arithmetic and the
same transforms in the same operation order; the integer streams are
bit-identical, the float transforms (log, cos, exp) may differ from the
device's libm by an ulp, so the checks allow 1 fp32 ulp after rounding."""

from __future__ import annotations

import numpy as np

M0, M1, W0, W1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57), 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox_raw(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 (Salmon et al., SC'11) of uint64-held 32-bit counter
    words (arrays) under key (k0, k1)."""
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return c0, c1, c2, c3


def philox(index, stream: int, seed: int):
    """Philox4x32-10 of counters (index lo, index hi, stream, 0), key = seed."""
    index = np.asarray(index, dtype=np.uint64)
    c0 = index & MASK
    c1 = index >> np.uint64(32)
    c2 = np.full_like(index, np.uint64(stream))
    c3 = np.zeros_like(index)
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    return philox_raw(c0, c1, c2, c3, k0, k1)


def u53(a, b):
    v = ((a >> np.uint64(5)) << np.uint64(26)) | (b >> np.uint64(6))
    return (v.astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def normal01(index, stream, seed):
    x0, x1, x2, x3 = philox(index, stream, seed)
    return np.sqrt(-2.0 * np.log(u53(x0, x1))) * np.cos(6.283185307179586 * u53(x2, x3))


def _fp32(r):
    r = np.clip(r, 1e-6, 1.0)
    return np.clip(r.astype(np.float32).astype(np.float64), 1e-6, 1.0)


def latent(user0, users, n, d, bias_kind, bias_scale, seed, quantize=True):
    sc = 1.0 / np.sqrt(float(d))
    P = normal01(np.arange(user0 * d, (user0 + users) * d, dtype=np.uint64), 1, seed).reshape(users, d) * sc
    Q = normal01(np.arange(n * d, dtype=np.uint64), 2, seed).reshape(n, d) * sc
    b = np.zeros(n)
    if bias_kind == 1:
        b = normal01(np.arange(n, dtype=np.uint64), 3, seed) * bias_scale
    elif bias_kind == 2:
        b = np.exp(normal01(np.arange(n, dtype=np.uint64), 3, seed) * bias_scale)
        part = np.zeros(256)
        for t in range(256):
            acc = 0.0
            for v in b[t::256]:
                acc += v
            part[t] = acc
        tot = 0.0
        for v in part:
            tot += v
        b = b - tot / n
    z = np.zeros((users, n))
    for c in range(d):
        z = z + P[:, c:c + 1] * Q[None, :, c]
    z = z + b[None, :]
    r = np.clip(1.0 / (1.0 + np.exp(-z)), 1e-6, 1.0)
    return _fp32(r) if quantize else r


def sparse(user0, users, n, per_user, zipf_s, floor_value, seed, quantize=True):
    k0, k1, _, _ = philox(np.arange(n, dtype=np.uint64), 4, seed)
    keys = (k0 << np.uint64(32)) | k1
    rank = np.empty(n)
    rank[np.argsort(keys, kind="stable")] = np.arange(1, n + 1)
    logp = -zipf_s * np.log(rank)
    out = np.full((users, n), floor_value)
    for ul in range(users):
        u = user0 + ul
        x0, x1, _, _ = philox(np.arange(u * n, (u + 1) * n, dtype=np.uint64), 5, seed)
        g = logp - np.log(-np.log(u53(x0, x1)))
        order = sorted(range(n), key=lambda i: (-g[i], i))[:per_user]
        for j, i in enumerate(order):
            base = (u * per_user + j) * 4
            l = []
            for c in range(4):
                y0, y1, y2, y3 = philox(np.array([base + c], dtype=np.uint64), 6, seed)
                l += [np.log(u53(y0, y1))[0], np.log(u53(y2, y3))[0]]
            g2 = -(l[0] + l[1])
            g5 = -((((l[2] + l[3]) + l[4]) + l[5]) + l[6])
            out[ul, i] = g2 / (g2 + g5)
    out = np.clip(out, 1e-6, 1.0)
    return _fp32(out) if quantize else out
