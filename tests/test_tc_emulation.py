"""Numerics of the tensor-core LWPR (csrc/lwpr_tc.cuh, the default LWPR kernel for
shared-metric models), emulated in numpy: the 3xTF32 logit GEMM -> exp -> a 3xTF32
moment GEMM P.V (the FlashAttention-shaped form; the kernel keeps the moments on
the CUDA cores, the emulation also covers moving them onto the tensor cores) stays
within 1e-5 absolute of the reference's float32 fast path on realistic rollout rows,
i.e. within the cost gate.  The GPU parity suite checks the kernel itself."""

import numpy as np

from oracle import rng
from oracle import rollout as RO
from oracle.lwpr import fold, predict_f32
from paper_1503_00330_b200 import synthetic


def tf32(a):
    b = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x0FFF + ((b >> 13) & 1)) & ~np.uint64(0x1FFF)  # round to nearest even, 10-bit mantissa
    return b.astype(np.uint32).view(np.float32)


def mm3(A, B):
    """3xTF32: hi*hi + hi*lo + lo*hi, products exact, float32 result per pass."""
    ah, bh = tf32(A), tf32(B)
    al, bl = tf32(np.float32(A) - ah), tf32(np.float32(B) - bh)
    f = lambda x, y: (x.astype(np.float64) @ y.astype(np.float64)).astype(np.float32)
    return f(ah, bh) + f(ah, bl) + f(al, bh)


def tc_predict(st, X):
    c, D, coef, lv = st.centers, st.metrics[0], st.coefs, st.lvar
    L = len(c)
    log2e = 1.4426950408889634
    mu = c.mean(0)
    ct, xt = c - mu, X.astype(np.float64) - mu
    dc = ct @ D.T
    a0 = -0.5 * np.einsum("ld,ld->l", dc, ct)
    q = -0.5 * np.einsum("bi,ij,bj->b", xt, D, xt)
    F = np.concatenate([xt, np.ones((len(X), 1)), q[:, None]], 1).astype(np.float32)
    W = (np.concatenate([dc.T, a0[None], np.ones((1, L))], 0) * log2e).astype(np.float32)
    P = np.exp2(mm3(F, W) + np.float32(64)).astype(np.float32)
    s = coef[:, 1:]
    y0 = coef[:, 0] - np.einsum("ld,ld->l", s, ct)
    g0, gs = y0.mean(), s.mean(0)
    y0s, ss = y0 - g0, s - gs
    cols = [np.ones(L), y0s, *ss.T, lv, y0s ** 2, *(2 * y0s * ss.T)]
    cols += [ss[:, i] * ss[:, j] * (1 if i == j else 2) for i in range(4) for j in range(i, 4)]
    Mo = mm3(P, np.stack(cols, 1).astype(np.float32)).astype(np.float64)
    den, x = Mo[:, 0], xt
    num = Mo[:, 1] + np.einsum("bi,bi->b", Mo[:, 2:6], x)
    quad = Mo[:, 7] + np.einsum("bi,bi->b", Mo[:, 8:12], x)
    k = 12
    for i in range(4):
        for j in range(i, 4):
            quad += Mo[:, k] * x[:, i] * x[:, j]
            k += 1
    mp = num / den
    return (g0 + x @ gs + mp).astype(np.float32), np.maximum((quad + Mo[:, 6]) / den - mp * mp, 0)


def test_three_pass_tf32_lwpr_within_gate():
    stacks = synthetic.hybrid_stacks(100, seed=0)
    K, N = 256, 50
    d = RO.Dyn()
    lo, hi = d.bounds()
    u = np.clip(np.tile([0, 0, 0, d.hover_thrust], (N, 1))[None] + rng.control_noise(0, 0, 0, K, N,
                                                                                      (2, 2, 0.8, 0.05)), lo, hi)
    ang, rate, xs = np.zeros((K, 3)), np.zeros((K, 3)), []
    for t in range(N):
        xs.append(np.concatenate([ang, u[:, t, 3:4]], 1))
        ang, rate = RO.wrap(ang + rate * d.dt), rate + 0.5 * (u[:, t, :3] - rate)
    X = np.stack(xs, 1).reshape(-1, 4).astype(np.float32)
    for a in range(3):
        rm, rv = predict_f32(fold(stacks[a].centers, stacks[a].metrics, stacks[a].coefs, stacks[a].lvar), X)
        tm, tv = tc_predict(stacks[a], X)
        assert np.abs(tm - rm).max() < 1e-5 * max(1.0, np.abs(rm).max())
        assert np.abs(np.sqrt(tv) - np.sqrt(rv)).max() / np.sqrt(rv).min() < 1e-4
