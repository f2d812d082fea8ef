"""LWPR models for the rollout engine (API of reference ``lwpr.py``).

``LwprModel`` / ``ReceptiveField`` hold a trained model's receptive fields
(lwpr.py:62-150); ``save_model`` / ``load_model`` read and write the
reference's "LWPR1" persistence format (lwpr.py:261-323) so a model trained
with the reference stages straight onto the GPU.  ``FrozenLwpr`` is the
drop-in for the reference's float32 fast path (lwpr.py:329-407): the same
constructor and ``predict_into(X, out_mean, out_var)``, evaluated by the
batched CUDA LWPR kernel.  Online training (RLS ``update``, lwpr.py:208-255)
is offline work outside the control step and is not part of this package.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from . import _abi

MAGIC = "LWPR1"


class LwprFormatError(ValueError):
    """Malformed persistence payload; carries a byte offset (lwpr.py:27-32)."""

    def __init__(self, message: str, offset: int = 0):
        super().__init__(f"{message} (at byte offset {offset})")
        self.offset = offset


@dataclass
class ReceptiveField:
    center: np.ndarray
    metric: np.ndarray
    coef: np.ndarray
    local_variance: float = 0.0
    var_acc: float = 0.0
    weight_count: float = 0.0
    inv_gram: np.ndarray = field(default=None)


def _metric_of(d_init, dim: int) -> np.ndarray:
    """d_init as a (dim, dim) metric: scalar -> scaled identity, vector -> diagonal,
    matrix -> its symmetric part (the reference's normalisation, lwpr.py:35-50)."""
    d = np.asarray(d_init, float)
    if d.ndim == 0:
        return float(d) * np.eye(dim)
    if d.shape == (dim,):
        return np.diag(d)
    if d.shape == (dim, dim):
        return 0.5 * (d + d.T)
    if d.ndim == 1:
        raise ValueError(f"d_init vector must have length {dim}")
    raise ValueError(f"d_init must be scalar, ({dim},) or ({dim},{dim})")


class LwprModel:
    """Receptive-field container with the reference's constructor (lwpr.py:100-124:
    same keywords, defaults and validation) and stacking accessor.  The
    hyperparameters only matter to training, which stays on the host in the
    reference; here they are carried for persistence (``save_model``)."""

    def __init__(self, input_dim: int, w_gen: float = 0.1, d_init=1.0, forgetting: float = 1.0,
                 ridge: float = 1e-3, participation: float = 1e-3):
        if input_dim < 1:
            raise ValueError("input_dim must be >= 1")
        if not 0.0 < w_gen < 1.0:
            raise ValueError("w_gen must be in (0, 1)")
        if not 0.0 < forgetting <= 1.0:
            raise ValueError("forgetting must be in (0, 1]")
        if ridge < 0.0:
            raise ValueError("ridge must be >= 0")
        self.input_dim = int(input_dim)
        self.w_gen = float(w_gen)
        self.d_init = _metric_of(d_init, self.input_dim)
        self.forgetting = float(forgetting)
        self.ridge = float(ridge)
        self.participation = float(participation)
        self.fields: list[ReceptiveField] = []
        self._stacked = None

    @property
    def hyperparams(self) -> dict:
        return {"w_gen": self.w_gen, "d_init": self.d_init, "forgetting": self.forgetting, "ridge": self.ridge,
                "participation": self.participation}

    @classmethod
    def from_stack(cls, centers, metrics, coefs, lvar) -> "LwprModel":
        centers = np.asarray(centers, float)
        m = cls(centers.shape[1])
        d = centers.shape[1]
        for i in range(centers.shape[0]):
            m.fields.append(ReceptiveField(centers[i].copy(), np.asarray(metrics[i], float).copy(),
                                           np.asarray(coefs[i], float).copy(), float(lvar[i]),
                                           inv_gram=np.eye(d + 1)))
        return m

    @property
    def num_fields(self) -> int:
        return len(self.fields)

    def _stacks(self):
        if self._stacked is None:
            self._stacked = stacks_of(self)
        return self._stacked


def stacks_of(model):
    """(centers (L,d), metrics (L,d,d), coefs (L,d+1), lvar (L,)) float64 of any LWPR model
    exposing ``fields`` (this package's or the reference's ``LwprModel``)."""
    fields = list(model.fields)
    if not fields:
        raise ValueError("no receptive fields")
    return (
        np.ascontiguousarray(np.stack([np.asarray(f.center, float) for f in fields])),
        np.ascontiguousarray(np.stack([np.asarray(f.metric, float) for f in fields])),
        np.ascontiguousarray(np.stack([np.asarray(f.coef, float) for f in fields])),
        np.ascontiguousarray(np.array([float(f.local_variance) for f in fields])),
    )


def save_model(model: LwprModel) -> bytes:
    """Serialise in the reference's "LWPR1" format (lwpr.py:261-285)."""
    d = model.input_dim
    hp = {k: getattr(model, k) for k in ("w_gen", "d_init", "forgetting", "ridge", "participation")
          if hasattr(model, k)}
    payload = {
        "input_dim": d,
        "hyperparams": {
            "w_gen": hp.get("w_gen", 0.1),
            "d_init": np.asarray(hp.get("d_init", np.eye(d)), float).tolist(),
            "forgetting": hp.get("forgetting", 1.0),
            "ridge": hp.get("ridge", 1e-3),
            "participation": hp.get("participation", 1e-3),
        },
        "fields": [
            {
                "center": np.asarray(f.center, float).tolist(),
                "metric": np.asarray(f.metric, float).tolist(),
                "coef": np.asarray(f.coef, float).tolist(),
                "local_variance": float(f.local_variance),
                "var_acc": float(f.var_acc),
                "weight_count": float(f.weight_count),
                "inv_gram": (np.eye(d + 1) if f.inv_gram is None else np.asarray(f.inv_gram, float)).tolist(),
            }
            for f in model.fields
        ],
    }
    return (MAGIC + "\n" + json.dumps(payload, sort_keys=True)).encode()


def load_model(data: bytes) -> LwprModel:
    """Parse an "LWPR1" payload (lwpr.py:288-323); raises LwprFormatError."""
    header = MAGIC.encode() + b"\n"
    if not data.startswith(header):
        raise LwprFormatError("bad magic header", offset=0)
    off = len(header)
    try:
        payload = json.loads(data[off:].decode())
    except (json.JSONDecodeError, UnicodeDecodeError) as e:
        raise LwprFormatError(f"invalid payload: {e}", offset=off + getattr(e, "pos", 0)) from e
    try:
        hp = payload["hyperparams"]
        model = LwprModel(int(payload["input_dim"]), w_gen=float(hp["w_gen"]),
                          d_init=np.array(hp["d_init"], dtype=np.float64), forgetting=float(hp["forgetting"]),
                          ridge=float(hp["ridge"]), participation=float(hp["participation"]))
        for fd in payload["fields"]:
            model.fields.append(ReceptiveField(
                center=np.array(fd["center"], dtype=np.float64),
                metric=np.array(fd["metric"], dtype=np.float64),
                coef=np.array(fd["coef"], dtype=np.float64),
                local_variance=float(fd["local_variance"]),
                var_acc=float(fd["var_acc"]),
                weight_count=float(fd["weight_count"]),
                inv_gram=np.array(fd["inv_gram"], dtype=np.float64),
            ))
    except (KeyError, TypeError, ValueError) as e:
        raise LwprFormatError(f"incomplete payload: {e}", offset=off) from e
    return model


def stage_axis(ctx: "_abi.Context", axis: int, model) -> None:
    """Fold one model's fields into the device layout (FrozenLwpr ctor, lwpr.py:339-358)."""
    c, m, k, v = stacks_of(model)
    L, d = c.shape
    ctx.call("pi2_set_lwpr_axis", int(axis), int(L), int(d), _abi.ptr(c), _abi.ptr(m), _abi.ptr(k),
             _abi.ptr(v))


class FrozenLwpr:
    """GPU drop-in for the reference's float32 fast path (lwpr.py:329-407).

    ``predict_into(X, out_mean, out_var=None)`` runs the batched CUDA LWPR
    kernel on float32 rows X (B, input_dim), B <= batch_rows.
    """

    def __init__(self, model, batch_rows: int, device: int = 0):
        if not model.fields:
            raise ValueError("no receptive fields")
        self.input_dim = int(model.input_dim)
        self.batch_rows = int(batch_rows)
        self._ctx = _abi.Context(device, 1, 1, 1)
        stage_axis(self._ctx, 0, model)

    def predict_into(self, X, out_mean, out_var=None) -> None:
        X = np.ascontiguousarray(X, dtype=np.float32)
        if X.ndim != 2 or X.shape[1] != self.input_dim:
            raise ValueError(f"X must have shape (B, {self.input_dim})")
        b = X.shape[0]
        if b > self.batch_rows:
            raise ValueError("more rows than the batch size given at construction")
        mean = np.empty(b, np.float32)
        var = np.empty(b, np.float32) if out_var is not None else None
        self._ctx.call("pi2_lwpr_predict", 0, int(b), _abi.ptr(X), _abi.ptr(mean), _abi.ptr(var))
        out_mean[...] = mean
        if out_var is not None:
            out_var[...] = var
