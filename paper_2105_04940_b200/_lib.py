"""ctypes binding of the C ABI (include/blockmm_b200.h) plus device plumbing.

The shared library is built in-tree (``python -m paper_2105_04940_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing, or no CUDA device is present, every compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
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
    "bmm_plan_small": (_I, [_I, _P, _P, _I64, _P, _P, _I64, _I64, _P, _P, _I, _P, _I64, _P, _I64] + [_P] * 18 + [_P]),
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
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)
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


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def want_numpy(*xs) -> bool:
    return not any(isinstance(x, torch.Tensor) for x in xs)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")
