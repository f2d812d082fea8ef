"""LWPR prediction restated from reference ``lwpr.py`` (test infrastructure only).

``fold`` is the parameter folding of ``FrozenLwpr.__init__``
(lwpr.py:339-358); ``predict_f32`` is ``FrozenLwpr.predict_into``
(lwpr.py:369-407) with the same numpy operation sequence (two small
sgemms, float32 exp, pairwise row sums), so results are bitwise equal to
the reference on the same numpy/OpenBLAS build.  ``predict_f64`` is the
float64 ``LwprModel.predict_batch`` (lwpr.py:185-203) and ``blend_loop``
the scalar-loop oracle of the reference tests (tests/oracles.py:16-44).
"""

from __future__ import annotations

import math

import numpy as np


def fold(centers, metrics, coefs, lvar) -> dict:
    """Fold one axis' receptive fields into float32 GEMM operands — lwpr.py:339-358."""
    centers = np.asarray(centers, np.float64)
    metrics = np.asarray(metrics, np.float64)
    coefs = np.asarray(coefs, np.float64)
    nf = centers.shape[0]
    if nf == 0:
        raise ValueError("no receptive fields")
    dc = np.einsum("lde,le->ld", metrics, centers)                      # :344
    p = {
        "a1": (-0.5 * np.einsum("ldd->ld", metrics)).T.astype(np.float32).copy(),  # :345
        "a2": dc.T.astype(np.float32).copy(),                                       # :346
        "a0": (-0.5 * np.einsum("ld,ld->l", dc, centers)).astype(np.float32),      # :347
    }
    off = metrics - metrics * np.eye(metrics.shape[1])[None]            # :348
    p["diagonal"] = bool(np.all(off == 0.0))                            # :349
    if not p["diagonal"]:                                               # :350-353
        p["axx"] = (-0.5 * metrics.reshape(nf, -1)).T.astype(np.float32).copy()
        p["a2f"] = dc.T.astype(np.float32).copy()
    p["slopes"] = coefs[:, 1:].T.astype(np.float32).copy()              # :354
    p["y0"] = (coefs[:, 0] - np.einsum("ld,ld->l", coefs[:, 1:], centers)).astype(np.float32)  # :355-357
    p["lvar"] = np.asarray(lvar, np.float64).astype(np.float32)         # :358
    return p


def predict_f32(p: dict, X: np.ndarray, want_var: bool = True):
    """Batched float32 mean/variance — lwpr.py:369-407 (fresh temporaries per call)."""
    X = np.asarray(X, np.float32)
    b, d = X.shape
    if p["diagonal"]:                                                   # :383-386
        q = np.matmul(np.multiply(X, X), p["a1"])
        t = np.matmul(X, p["a2"])
    else:                                                               # :387-392
        xq = np.multiply(X[:, :, None], X[:, None, :]).reshape(b, d * d)
        q = np.matmul(xq, p["axx"])
        t = np.matmul(X, p["a2f"])
    q += t                                                              # :393
    q += p["a0"][None, :]                                               # :394
    np.exp(q, out=q)                                                    # :395
    den = q.sum(axis=1)                                                 # :396
    q /= den[:, None]                                                   # :397
    y = np.matmul(X, p["slopes"])                                       # :398
    y += p["y0"][None, :]                                               # :399
    np.multiply(q, y, out=t)                                            # :400
    mean = t.sum(axis=1)                                                # :401
    if not want_var:
        return mean, None
    np.subtract(mean[:, None], y, out=t)                                # :403
    np.multiply(t, t, out=t)                                            # :404
    t += p["lvar"][None, :]                                             # :405
    t *= q                                                              # :406
    return mean, t.sum(axis=1)                                          # :407


def predict_f64(centers, metrics, coefs, lvar, X):
    """Float64 blended mean/variance — lwpr.py:185-203."""
    X = np.asarray(X, np.float64)
    diff = X[:, None, :] - np.asarray(centers)[None, :, :]
    quad = np.einsum("bld,lde,ble->bl", diff, np.asarray(metrics), diff)
    w = np.exp(-0.5 * quad)
    w /= w.sum(axis=1, keepdims=True)
    coefs = np.asarray(coefs)
    y = coefs[None, :, 0] + np.einsum("bld,ld->bl", diff, coefs[:, 1:])
    mean = (w * y).sum(axis=1)
    dev = mean[:, None] - y
    return mean, (w * (dev * dev + np.asarray(lvar)[None, :])).sum(axis=1)


def blend_loop(centers, metrics, coefs, lvar, x):
    """Scalar-loop Eq. 1 with math.exp (reference tests/oracles.py:16-44)."""
    raw, preds = [], []
    for j in range(len(centers)):
        d = [x[k] - centers[j][k] for k in range(len(x))]
        quad = sum(d[a] * metrics[j][a][b] * d[b] for a in range(len(x)) for b in range(len(x)))
        raw.append(math.exp(-0.5 * quad))
        preds.append(coefs[j][0] + sum(coefs[j][1 + k] * d[k] for k in range(len(x))))
    tot = sum(raw)
    w = [r / tot for r in raw]
    mean = sum(wi * pi for wi, pi in zip(w, preds))
    var = sum(wi * ((mean - pi) ** 2 + s) for wi, pi, s in zip(w, preds, lvar))
    return mean, var


def hybrid_eval(folded_axes, X, want_std: bool):
    """``HybridModel.make_batch_eval`` → eval_into — dynamics.py:262-277."""
    X = np.asarray(X, np.float32)
    mean = np.empty((X.shape[0], 3), np.float32)
    std = np.empty((X.shape[0], 3), np.float32) if want_std else None
    for axis in range(3):
        m, v = predict_f32(folded_axes[axis], X, want_std)
        mean[:, axis] = m
        if want_std:
            std[:, axis] = v
    if want_std:
        np.sqrt(std, out=std)                                            # :274-275
    return mean, std


def analytic_eval(X, mass, gravity, want_std: bool):
    """``AnalyticModel.make_batch_eval`` → eval_into — dynamics.py:166-187."""
    X = np.asarray(X, np.float32)
    inv_m = np.float32(1.0 / mass)
    g = np.float32(gravity)
    sr, cr = np.sin(X[:, 0]), np.cos(X[:, 0])
    sp, cp = np.sin(X[:, 1]), np.cos(X[:, 1])
    sy, cy = np.sin(X[:, 2]), np.cos(X[:, 2])
    fm = X[:, 3] * inv_m
    mean = np.empty((X.shape[0], 3), np.float32)
    mean[:, 0] = fm * (cr * sp * cy + sr * sy)
    mean[:, 1] = fm * (cr * sp * sy - sr * cy)
    mean[:, 2] = fm * (cr * cp) - g
    std = np.zeros((X.shape[0], 3), np.float32) if want_std else None
    return mean, std
