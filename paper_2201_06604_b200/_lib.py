"""ctypes binding of libsfb.so (include/sfb.h) -- the only way into the kernels.

There is deliberately no fallback: if the shared library is missing or was not
built for sm_100a, every device entry point raises.  (The reference's own CPU
path lives only in oracle/, which this package never imports.)
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# SFB_LIB: load another build of the library (A/B timing of kernel changes only)
LIB_PATH = os.environ.get("SFB_LIB") or os.path.join(_HERE, "libsfb.so")

SFB_F64, SFB_F32, SFB_I64 = 0, 1, 2

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int

_SIGS = {
    "sfb_last_error": ([], ctypes.c_char_p),
    "sfb_version": ([], _int),
    "sfb_device_ok": ([], _int),
    "sfb_host_register": ([_vp, _i64], _int),
    "sfb_host_unregister": ([_vp], _int),
    "sfb_validate_seed": ([_i64p], _int),
    "sfb_next_state": ([_i64p, _i64p], _int),
    "sfb_jump_matrices": ([_int, _i64p, _i64p], _int),
    "sfb_jump_ahead": ([_i64p, _int], _int),
    "sfb_skip": ([_i64p, ctypes.c_uint64], _int),
    "sfb_create_streams": ([_i64p, _i64, _i64p, _i64p], _int),
    "sfb_format_streams_bound": ([_i64], _i64),
    "sfb_format_streams": ([_i64p, _i64p, _i64, ctypes.c_char_p, _i64, _i64p], _int),
    "sfb_save_streams": ([ctypes.c_char_p, _i64p, _i64p, _i64, _int], _int),
    "sfb_parse_streams_count": ([ctypes.c_char_p, _i64, _i64p], _int),
    "sfb_parse_streams": ([ctypes.c_char_p, _i64, _i64p, _i64p, _i64], _int),
    "sfb_fill_real": ([_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _int, ctypes.c_double,
                       _i64, _i64, _int, _vp], _int),
    "sfb_fill_integer": ([_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _int, _vp],
                         _int),
    "sfb_fill_normal": ([_vp, _i64, _vp, _int, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _int,
                         _vp], _int),
    "sfb_fisher_replicates": ([_vp, _i64, _i64p, _int, _i64p, _int, _f64p, _i64,
                               ctypes.c_double, _i64, _i64, _i64, _vp, _vp, _vp, _int, _vp],
                              _int),
    "sfb_fisher_replicates_host": ([_vp, _i64, _i64p, _int, _i64p, _int, _f64p, _i64,
                                    ctypes.c_double, _i64, _i64, _i64, _vp, _vp, _vp], _int),
    "sfb_rcont2_table": ([_i64p, _int, _i64p, _int, _f64p, _i64, _vp, _vp, _vp], _int),
    "sfb_fisher_memo_pending": ([], _int),
    "sfb_probe_fp64": ([_vp, _i64, _int, _vp], _int),
    "sfb_probe_dmma": ([_vp, _i64, _int, _vp], _int),
    "sfb_probe_rsqrt": ([_vp, _vp, _i64, _vp], _int),
    "sfb_bessel_k": ([ctypes.c_double, _vp, _i64, _vp, _vp], _int),
    "sfb_matern_correlation": ([ctypes.c_double, ctypes.c_double, _vp, _i64, _vp, _vp], _int),
    "sfb_matern_cov": ([_f64p, _int, _vp, _i64, _int, _int, ctypes.c_double, _vp, _vp, _vp], _int),
    "sfb_matern_scratch_bytes": ([_int, _int, _int], _i64),
    "sfb_host_bessel_k": ([ctypes.c_double, ctypes.c_double], ctypes.c_double),
    "sfb_chol_batch": ([_vp, _i64, _i64, _vp, _vp, _vp, _vp], _int),
    "sfb_lower_diag_multiply": ([_vp, _vp, _i64, _i64, _vp, _int, _i64, _int, _vp, _vp], _int),
    "sfb_download_shard": ([_vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _vp], _int),
    "sfb_probe_write": ([_vp, _i64, _int, _vp], _int),
    "sfb_host_step_u32": ([_i64p, _i64, _i64, _i64p], _int),
    "sfb_host_exp": ([ctypes.c_double], ctypes.c_double),
    "sfb_host_log1p": ([ctypes.c_double], ctypes.c_double),
    "sfb_host_log1p_fill": ([ctypes.c_double, ctypes.POINTER(ctypes.c_int)], ctypes.c_double),
    "sfb_host_box_muller": ([_i64p, _i64p, _i64, _f64p, _f64p], _int),
    "sfb_host_box_muller_f32": ([_i64p, _i64p, _i64, _int, ctypes.c_double, _f32p, _f32p], _int),
    "sfb_host_fisher_replicates": ([_i64p, _i64p, _int, _i64p, _int, _f64p, ctypes.c_double,
                                    _i64, _i64, _i64, _f64p, _i64p], _int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libsfb.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().sfb_last_error().decode(errors="replace")
        raise errors.from_status(rc, msg)


def ptr(a, t=_i64p):
    """ctypes pointer to a numpy array's buffer."""
    return a.ctypes.data_as(t)


def dptr(t) -> int:
    """raw device address of a torch tensor."""
    return t.data_ptr()


# device -> numpy through a pinned block of torch's caching host allocator:
# one DMA at PCIe speed (a fresh pageable .cpu() runs at ~2 GB/s: page faults
# plus a staged copy; 800 MB: 400 ms vs 15 ms once the block is cached).
# Above this size the array stays pageable (pinned blocks stay cached).
PINNED_HOST_MAX = 4 << 30


def to_host(t) -> np.ndarray:
    """numpy copy of a CUDA tensor (synchronous)."""
    import torch

    nbytes = t.numel() * t.element_size()
    if t.is_cuda and 0 < nbytes <= PINNED_HOST_MAX:
        try:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        except RuntimeError:
            return t.cpu().numpy()
        h.copy_(t)
        return h.numpy()
    return t.cpu().numpy()


_DEVICE_OK = False


def require_device():
    """The product path needs an sm_100a GPU; fail loudly otherwise (the
    positive answer is cached: it is asked on every API call)."""
    global _DEVICE_OK
    if _DEVICE_OK:
        return
    import torch

    if not torch.cuda.is_available():
        raise errors.DeviceError("no CUDA device visible: the B200 kernels have no CPU fallback")
    if not lib().sfb_device_ok():
        raise errors.DeviceError("libsfb.so is built for sm_100a only (B200); this device is not")
    _DEVICE_OK = True


def stream_handle():
    """cudaStream_t of torch's current stream on the current device (the raw
    query costs ~0.1 us; building a torch.cuda.Stream object ~3 us)."""
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream
