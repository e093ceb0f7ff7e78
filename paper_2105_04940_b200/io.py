"""Wire and on-disk formats -- SURVEY.md §8(f4).

* matrix binary (matrix.py:121-140): ``<QQ`` little-endian rows, cols, then the
  row-major float64-LE payload.  ``load_matrix(path, device=True)`` streams the
  payload straight into a CUDA tensor through a pinned staging buffer in
  chunks (no intermediate pageable copy of the whole matrix), so a large
  instance lands in HBM at PCIe rate; ``save_matrix`` accepts CUDA tensors and
  writes them the same way in reverse.
* matrix CSV (matrix.py:143-159): one row per line, ``%.17g``.
* instance sidecar (datagen.py:113-140): two binary matrices + sorted JSON.
* plan JSON and SampleLog CSV live with their types (plan.py, estimators.py).

Byte-identical to the reference's writers; the readers return what the
reference's return (tests/test_io.py against files written by the reference).
"""
from __future__ import annotations

import csv
import json
import os
import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .matrix import as_matrix

_HEADER = struct.Struct("<QQ")
_CHUNK = 64 << 20  # staging chunk, bytes


def _check_finite_device(t: torch.Tensor) -> None:
    if not bool(torch.isfinite(t).all().item()):
        raise ValueError("matrix contains NaN or Inf entries")


def save_matrix(path, M) -> None:
    """matrix.py:121-127; CUDA tensors are staged through pinned memory."""
    if isinstance(M, torch.Tensor) and M.device.type == "cuda":
        if M.ndim != 2:
            raise ValueError(f"expected a 2-D matrix, got ndim={M.ndim}")
        t = M.to(torch.float64).contiguous()
        _check_finite_device(t)
        rows, cols = t.shape
        flat = t.view(-1)
        stage = torch.empty(min(flat.numel(), _CHUNK // 8) or 1, dtype=torch.float64).pin_memory()
        with open(path, "wb") as f:
            f.write(_HEADER.pack(rows, cols))
            for s in range(0, flat.numel(), stage.numel()):
                e = min(flat.numel(), s + stage.numel())
                stage[:e - s].copy_(flat[s:e])
                f.write(stage[:e - s].numpy().astype("<f8", copy=False).tobytes())
        return
    a = as_matrix(M.cpu().numpy() if isinstance(M, torch.Tensor) else M)
    with open(path, "wb") as f:
        f.write(_HEADER.pack(a.shape[0], a.shape[1]))
        f.write(a.astype("<f8", copy=False).tobytes(order="C"))


def load_matrix(path, device: bool = False):
    """matrix.py:130-140.  device=True returns a CUDA float64 tensor, read
    chunk-wise into pinned memory and copied asynchronously (double buffered)."""
    path = Path(path)
    size = os.path.getsize(path)
    if size < _HEADER.size:
        raise ValueError(f"{path}: truncated header")
    with open(path, "rb") as f:
        rows, cols = _HEADER.unpack(f.read(_HEADER.size))
        expected = _HEADER.size + rows * cols * 8
        if size != expected:
            raise ValueError(f"{path}: expected {expected} bytes, found {size}")
        if not device:
            payload = np.frombuffer(f.read(), dtype="<f8")
            return as_matrix(payload.reshape(rows, cols))
        out = torch.empty((rows, cols), dtype=torch.float64, device=_lib.device())
        flat = out.view(-1)
        total = rows * cols
        per = max(1, min(total, _CHUNK // 8))
        stages = [torch.empty(per, dtype=torch.float64).pin_memory() for _ in range(2)]
        events = [None, None]
        stream = torch.cuda.current_stream()
        for i, s in enumerate(range(0, total, per)):
            e = min(total, s + per)
            buf = stages[i & 1]
            if events[i & 1] is not None:
                events[i & 1].synchronize()  # the copy out of this buffer has finished
            view = buf[:e - s].numpy()
            got = f.readinto(memoryview(view).cast("B"))
            if got != (e - s) * 8:
                raise ValueError(f"{path}: short read")
            if view.dtype.byteorder == ">":  # pragma: no cover - big-endian host
                view.byteswap(inplace=True)
            flat[s:e].copy_(buf[:e - s], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            events[i & 1] = ev
        _check_finite_device(out)
        return out


def save_matrix_csv(path, M) -> None:
    """matrix.py:143-149."""
    a = as_matrix(M.cpu().numpy() if isinstance(M, torch.Tensor) else M)
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        for row in a:
            w.writerow(f"{x:.17g}" for x in row)


def load_matrix_csv(path) -> np.ndarray:
    """matrix.py:152-159."""
    with open(path, newline="") as f:
        rows = [[float(x) for x in line] for line in csv.reader(f) if line]
    if not rows:
        raise ValueError(f"{path}: empty CSV matrix")
    return as_matrix(np.array(rows))


def save_instance(prefix, M, N, metadata: dict) -> dict:
    """datagen.py:113-132: <prefix>_left.bin, <prefix>_right.bin, <prefix>.json."""
    prefix = Path(prefix)
    prefix.parent.mkdir(parents=True, exist_ok=True)
    left = prefix.with_name(prefix.name + "_left.bin")
    right = prefix.with_name(prefix.name + "_right.bin")
    save_matrix(left, M)
    save_matrix(right, N)
    doc = dict(metadata)
    doc.update(left_file=left.name, right_file=right.name, left_shape=list(M.shape), right_shape=list(N.shape))
    prefix.with_name(prefix.name + ".json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")
    return doc


def load_instance(prefix, device: bool = False):
    """datagen.py:135-140 (device=True: both factors straight into HBM)."""
    prefix = Path(prefix)
    doc = json.loads(prefix.with_name(prefix.name + ".json").read_text())
    M = load_matrix(prefix.with_name(doc["left_file"]), device=device)
    N = load_matrix(prefix.with_name(doc["right_file"]), device=device)
    if list(M.shape) != doc["left_shape"] or list(N.shape) != doc["right_shape"]:
        raise ValueError("stored shapes disagree with the sidecar")
    return M, N, doc
