"""Exact (bit-preserving) JSON encoding of numpy arrays and floats for golden fixtures."""

from __future__ import annotations

import base64
import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def enc(a) -> dict:
    a = np.ascontiguousarray(np.asarray(a))
    return {"dtype": str(a.dtype), "shape": list(a.shape), "b64": base64.b64encode(a.tobytes()).decode()}


def dec(d: dict) -> np.ndarray:
    raw = base64.b64decode(d["b64"])
    return np.frombuffer(raw, dtype=np.dtype(d["dtype"])).reshape(d["shape"]).copy()


def fhex(x: float) -> str:
    return float(x).hex()


def unhex(s: str) -> float:
    return float.fromhex(s)


def save(name: str, obj) -> Path:
    path = HERE / f"{name}.json"
    path.write_text(json.dumps(obj, separators=(",", ":")))
    return path


def load(name: str):
    return json.loads((HERE / f"{name}.json").read_text())
