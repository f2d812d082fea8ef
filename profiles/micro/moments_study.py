# profiles/micro/moments_study.py -- CPU only: python profiles/micro/moments_study.py
# Numerical study (CPU): second moment of the LWPR prediction as an expanded quadratic form
# (what a second tensor-core GEMM would produce) vs the direct e*(y'^2) form, both in float32,
# against float64.  Local models shifted by the mean local model g (as the kernel does).
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1503_00330_b200 import synthetic as S

st = S.hybrid_stacks(100, seed=0)
rng = np.random.default_rng(3)
X = rng.uniform(S.CENTER_LO - 0.1, S.CENTER_HI + 0.1, size=(200000, 4))
worst = {}
for ax, stack in enumerate(st):
    c, D, coef, lv = (np.asarray(a, np.float64) for a in (stack.centers, stack.metrics, stack.coefs, stack.lvar)) \
        if hasattr(stack, 'centers') else (np.asarray(a, np.float64) for a in stack)
    L = c.shape[0]
    mu = c.mean(0)
    slopes = coef[:, 1:]                    # (L, 4)
    y0 = coef[:, 0] - np.einsum('ld,ld->l', slopes, c)   # y_l(x) = y0_l + slopes_l . x
    g0, gs = y0.mean(), slopes.mean(0)      # mean local model g(x) = g0 + gs . x
    Xt = X - mu
    # shifted local models in centred coordinates: y'_l = Y0'_l + S'_l . x~
    Sp = slopes - gs
    Y0p = (y0 - g0) + Sp @ mu
    d = X[:, None, :] - c[None]
    q = 0.5 * np.einsum('bld,lde,ble->bl', d, D, d)
    e = np.exp(-(q - q.min(1, keepdims=True)))         # weights (row-normalised scale)
    yp = Y0p[None] + Xt @ Sp.T                          # (B, L) float64 truth
    den = e.sum(1); m1 = (e * yp).sum(1); m2 = (e * (yp * yp + lv[None])).sum(1)
    var64 = m2 / den - (m1 / den) ** 2
    f = np.float32
    e32, yp32 = e.astype(f), (Y0p.astype(f)[None] + Xt.astype(f) @ Sp.astype(f).T).astype(f)
    den32 = e32.sum(1, dtype=f)
    m1d = (e32 * yp32).sum(1, dtype=f); m2d = (e32 * (yp32 * yp32 + lv.astype(f)[None])).sum(1, dtype=f)
    var_direct = m2d / den32 - (m1d / den32) ** 2
    # expanded: sum e Y0'^2 + 2 x.(sum e Y0' S') + x^T (sum e S'S'^T) x + sum e lv, GEMM sums in float32
    A0 = e32 @ (Y0p * Y0p + lv).astype(f)
    A1 = e32 @ (Y0p[:, None] * Sp).astype(f)             # (B, 4)
    A2 = (e32 @ np.einsum('li,lj->lij', Sp, Sp).reshape(L, 16).astype(f)).reshape(-1, 4, 4)
    xt32 = Xt.astype(f)
    m2e = A0 + 2 * (xt32 * A1).sum(1, dtype=f) + np.einsum('bi,bij,bj->b', xt32, A2, xt32).astype(f)
    var_exp = m2e / den32 - (m1d / den32) ** 2
    sd64 = np.sqrt(np.maximum(var64, 0))
    for name, v in (('direct', var_direct), ('expanded', var_exp)):
        err = np.abs(np.sqrt(np.maximum(v, 0)) - sd64) / np.maximum(sd64, 1e-30)
        print(f"axis {ax} {name:9s}: std rel err max {err.max():.2e}  p99.9 {np.quantile(err, 0.999):.2e}")
