"""ctypes binding of the C ABI (include/blockmm_b200.h) plus device plumbing.

The shared library is built in-tree (``python -m paper_2105_04940_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing, or no CUDA device is present, every compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np
import torch

LIB_PATH = Path(__file__).resolve().parent / "libbmm_b200.so"

BMM_F64, BMM_F32 = 0, 1
RULE_EXPLICIT, RULE_ONC, RULE_OPL, RULE_TWO_STEP, RULE_UU, RULE_PILOT = 0, 1, 2, 3, 4, 5

ST_OK = 0
ST_ZERO_SCORE = 1
ST_CAUCHY_SCHWARZ = 2
ST_RADICAND = 3
ST_ALL_ZERO_WEIGHT = 4
ST_BAD_WEIGHT = 5
ST_CAP_BELOW_FLOOR = 6
ST_BELOW_FLOORS = 7
ST_ABOVE_CAPS = 8
ST_NO_CONVERGE = 9
ST_NOT_PLACED = 10
ST_EMPTY_SUPPORT = 11
ST_PLAN_MISMATCH = 12
ST_BAD_PROBS = 13

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int

# name -> (restype, argtypes); mirrors include/blockmm_b200.h
SIGNATURES = {
    "bmm_version": (_I, []),
    "bmm_last_error": (ctypes.c_char_p, []),
    "bmm_launch_count": (_I64, []),
    "bmm_copy2d": (_I, [_P, _I64, _P, _I64, _I64, _I64, _I, _P]),
    "bmm_norms": (_I, [_I, _P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I, _P, _P, _P]),
    "bmm_block_probs": (_I, [_P, _P, _I64, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P]),
    "bmm_normalize": (_I, [_P, _I64, _I64, _P, _P, _P]),
    "bmm_budgets_workspace": (_I64, [_I64]),
    "bmm_budgets": (_I, [_I, _P, _P, _P, _P, _P, _I64, _I64, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "bmm_block_cdf": (_I, [_P, _P, _I64, _I64, _I64, _P, _P, _P]),
    "bmm_seed_streams": (_I, [_P, _I64, _P, _I64, _I64, _P, _P]),
    "bmm_sample": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "bmm_sample_reps": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "bmm_compress_workspace": (_I64, [_I64, _I64]),
    "bmm_compress_sketch": (_I, [_P, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _P, _P]),
    "bmm_gemm_f64_dk": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P, _I64,
                             _P]),
    "bmm_gather": (_I, [_I, _I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I64, _I64,
                        _P, _I64, _I64, _P, _I64, _I64, _P]),
    "bmm_gather_dk": (_I, [_I, _I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I64, _P, _I64,
                           _P, _I64, _I64, _P, _I64, _I64, _P]),
    "bmm_gather_blocks": (_I, [_I, _P, _I64, _P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64,
                               _P, _I64, _P, _I64, _P]),
    "bmm_gemm_f64_workspace": (_I64, [_I64, _I64, _I64, _I64]),
    "bmm_gemm_f64_set_variant": (_I, [_I, _I]),
    "bmm_gemm_f64": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64,
                          _P, _I64, _P]),
    "bmm_gemm_f64_gather": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I64, _I64, _P,
                                 _I64, _I64, _P, _I64, _P]),
    "bmm_segsq_f64_gather": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _I64, _I64,
                                  _I64, _P, _P, _I64, _P]),
    "bmm_segsq_f64_workspace": (_I64, [_I64, _I64, _I64, _I64]),
    "bmm_segsq_f64": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P,
                           _P, _I64, _P]),
    "bmm_segsq_i8_workspace": (_I64, [_I64, _I64, _I64, _I64, _I64]),
    "bmm_segsq_i8": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P,
                          _P, _I64, _P]),
    "bmm_segsq_i8_timed": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P,
                                _P, _I64, _P, _P]),
    "bmm_gemm_i8_workspace": (_I64, [_I64, _I64, _I64, _I64]),
    "bmm_gemm_i8": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _I64, _I64,
                         _P, _I64, _P]),
    "bmm_gemm_i8_gather": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64,
                                _P, _I64, _I64, _P, _I64, _P]),
    "bmm_balance_exponents": (_I, [_P, _P, _I64, _P, _I64, _I64, _P, _I64, _P, _P]),
    "bmm_segsq_gram_gather": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _I64, _I64,
                                   _I64, _I64, _P, _P]),
    "bmm_segsq_gram_max_len": (_I64, []),
    "bmm_expand_blocks": (_I, [_P, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _I64, _P]),
    "bmm_segsq_gram": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P, _P]),
    "bmm_segsq_gram_norms": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P, _P, _P,
                                  _I64, _P]),
    "bmm_variance_workspace": (_I64, [_I64, _I64, _I64, _I64]),
    "bmm_elementwise_variance": (_I, [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _P, _P, _P, _I64,
                                      _P, _P, _I64, _P]),
    "bmm_block_term1": (_I, [_P, _P, _P, _P, _I64, _P, _P, _P]),
    "bmm_gen_instance": (_I, [_I, _I, _I64, _I64, _I64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                              ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, _P, _I64, _P,
                              _I64, _P]),
    "bmm_ar1_transform": (_I, [_I, _P, _I64, _I64, _I64, _I, ctypes.c_double, ctypes.c_double, _P, ctypes.c_double,
                               _P, _I64, _P]),
    "bmm_plan_small_smem": (_I64, [_I64, _I64, _I64]),
    "bmm_plan_small_debug": (_I, [_P]),
    "bmm_plan_small": (_I, [_I, _P, _P, _I64, _P, _P, _I64, _I64, _I64, _P, _P, _I, _P, _I64, _P, _I64] + [_P] * 18 + [_P]),
    "bmm_gemm_f64_err_workspace": (_I64, [_I64, _I64, _I64, _I64]),
    "bmm_gemm_f64_err": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64,
                              _P, _P, _I64, _P]),
    "bmm_sqdiff_workspace": (_I64, [_I64, _I64, _I64]),
    "bmm_sqdiff": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _P]),
    "bmm_pairwise_sum": (_I, [_P, _I64, _I64, _I64, _P, _P]),
    "bmm_gather_f32split": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I64, _I64,
                               _P, _P, _P, _P, _P]),
    "bmm_gather_f32split_dk": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I64, _P, _I64,
                                    _P, _P, _P, _P, _P]),
    "bmm_gemm_f32split_dk": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P]),
    "bmm_balance_f16": (_I, [_P, _P, _I64, _P, _P, _I64, _I64, _P, _I64, _P, _P, _P]),
    "bmm_gather_f16split_dk": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _P,
                                    _I64, _P, _P, _P, _P, _P]),
    "bmm_gemm_f16split_dk": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _I64, _P, _I64, _I64, _P]),
    "bmm_gemm_f32split": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _P]),
    "bmm_timestamp": (_I, [_P, _P]),
    "bmm_gemm_f32split_gather": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I64, _P, _I64,
                                      _P, _I64, _I64, _P]),
    "bmm_nccl_version": (_I, []),
    "bmm_nccl_unique_id": (_I, [_P]),
    "bmm_nccl_comm_init": (_I, [_P, _I, _P, _I]),
    "bmm_nccl_comm_destroy": (_I, [_P]),
    "bmm_all_gather_f64_nccl": (_I, [_P, _P, _I64, _P, _P]),
    "bmm_exchange_sum_nccl": (_I, [_P, _I, _P, _I64, _P, _P, _P]),
    "bmm_gemm_f16split_gather": (_I, [_I, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64,
                                      _P, _I64, _P, _I64, _I64, _P]),
}

_lib = None


class ExtensionMissing(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ExtensionMissing(
            f"{LIB_PATH} is missing: build it with `python -m paper_2105_04940_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2105_04940_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def call(name: str, *args) -> int:
    """Invoke a C-ABI entry point; negative return codes raise RuntimeError."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if isinstance(rc, int) and rc < 0 and SIGNATURES[name][0] is _I:
        msg = lib.bmm_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed ({rc}): {msg}")
    return rc


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def launches() -> int:
    return int(load().bmm_launch_count())


# ---------------------------------------------------------------- tensors

def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(x, dtype=None) -> torch.Tensor:
    """Host (numpy) or device tensor -> contiguous CUDA tensor, no copy when already there."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to(dev, non_blocking=True)
    else:
        a = np.asarray(x)
        t = _upload(np.ascontiguousarray(a))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_contiguous():
        t = t.contiguous()
    return t


def matrix_dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return BMM_F64
    if t.dtype == torch.float32:
        return BMM_F32
    raise TypeError(f"unsupported matrix dtype {t.dtype}")


def float_matrix(x) -> torch.Tensor:
    """CUDA float64/float32 matrix view of x (other dtypes are coerced to float64)."""
    t = to_device(x)
    if t.dtype not in (torch.float64, torch.float32):
        t = t.to(torch.float64)
    return t


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())


def i64(values) -> torch.Tensor:
    return torch.as_tensor(np.asarray(values, dtype=np.int64), device=device())


def f64(values) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64), device=device())


# ---- large host <-> device transfers of the drop-in API (numpy in, numpy out): pageable
# memory moves through two pinned staging buffers, the PCIe copy of one chunk overlapping the
# host-side memcpy of the other (4 threads; first-touch page faults of a fresh result array
# are what bound a plain `.cpu()`: config 4's C and D, 4.3 GB each).  Measured on the B200 box
# (tools/host_copy_probe.py, profiles/r2be_host_copy_probe.txt): plain copies are as fast up to
# 32 MB and fall to 2.2 GB/s (D2H) / 11 GB/s (H2D) from 64 MB on; staged 23 / 41 GB/s at 4.3 GB.
_BIG = 48 << 20
_CHUNK = 64 << 20
_stage = None
_stage_lock = threading.Lock()  # one staged transfer at a time: the two pinned buffers are shared


def _staging():
    global _stage
    if _stage is None:
        from concurrent.futures import ThreadPoolExecutor
        workers = max(2, min(8, (os.cpu_count() or 4) // 2))
        _stage = {"pin": [torch.empty(_CHUNK, dtype=torch.uint8).pin_memory() for _ in range(2)],
                  "stream": torch.cuda.Stream(), "pool": ThreadPoolExecutor(max_workers=workers), "workers": workers}
    return _stage


def _par_copy(pool, dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (flat uint8 views) on the pool's threads (numpy releases the GIL)."""
    n = dst.size
    parts = _stage["workers"]
    step = max(1, -(-n // parts))
    futs = [pool.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, n, step)]
    for f in futs:
        f.result()


def host(t: torch.Tensor) -> np.ndarray:
    t = t.detach()
    nbytes = t.numel() * t.element_size()
    if t.device.type != "cuda" or nbytes < _BIG or not t.is_contiguous():
        return t.cpu().numpy()
    with _stage_lock:
        return _host_staged(t, nbytes)


def _host_staged(t: torch.Tensor, nbytes: int) -> np.ndarray:
    sg = _staging()
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    dst = out.reshape(-1).view(np.uint8)
    src = t.reshape(-1).view(torch.uint8)
    cs = sg["stream"]
    cs.wait_stream(torch.cuda.current_stream())
    pend = None  # (event, offset, length, buffer index) of the chunk in flight
    for i, off in enumerate(range(0, nbytes, _CHUNK)):
        ln = min(_CHUNK, nbytes - off)
        buf = sg["pin"][i & 1]
        with torch.cuda.stream(cs):
            buf[:ln].copy_(src[off:off + ln], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        if pend is not None:
            pev, poff, pln, pi = pend
            pev.synchronize()
            _par_copy(sg["pool"], dst[poff:poff + pln], sg["pin"][pi].numpy()[:pln])
        pend = (ev, off, ln, i & 1)
    pev, poff, pln, pi = pend
    pev.synchronize()
    _par_copy(sg["pool"], dst[poff:poff + pln], sg["pin"][pi].numpy()[:pln])
    return out


def _upload(a: np.ndarray) -> torch.Tensor:
    """Contiguous numpy array -> CUDA tensor; large pageable arrays through the staging buffers."""
    dev = device()
    nbytes = a.nbytes
    th = torch.from_numpy(a)
    if nbytes < _BIG or th.is_pinned():
        return th.to(dev, non_blocking=False)
    with _stage_lock:
        return _upload_staged(a, th, dev, nbytes)


def _upload_staged(a: np.ndarray, th: torch.Tensor, dev, nbytes: int) -> torch.Tensor:
    sg = _staging()
    out = torch.empty(a.shape, dtype=th.dtype, device=dev)
    dst = out.reshape(-1).view(torch.uint8)
    src = a.reshape(-1).view(np.uint8)
    cs = sg["stream"]
    cs.wait_stream(torch.cuda.current_stream())
    evs = [None, None]
    for i, off in enumerate(range(0, nbytes, _CHUNK)):
        ln = min(_CHUNK, nbytes - off)
        if evs[i & 1] is not None:
            evs[i & 1].synchronize()  # the buffer's previous chunk has left for the device
        buf = sg["pin"][i & 1]
        _par_copy(sg["pool"], buf.numpy()[:ln], src[off:off + ln])
        with torch.cuda.stream(cs):
            dst[off:off + ln].copy_(buf[:ln], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        evs[i & 1] = ev
    torch.cuda.current_stream().wait_stream(cs)
    for ev in evs:
        if ev is not None:
            ev.synchronize()
    return out


def want_numpy(*xs) -> bool:
    return not any(isinstance(x, torch.Tensor) for x in xs)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")
