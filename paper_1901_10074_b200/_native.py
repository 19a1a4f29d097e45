"""ctypes binding of libhefv.so (the C-ABI in include/hefv.h).

There is no CPU fallback: importing the FV backend without the built
library, or without a CUDA device, raises ``NativeError`` immediately.
Device memory comes from torch's caching allocator; every call passes raw
device pointers plus the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import NativeError

_LIB_PATH = Path(os.environ.get("HEFV_LIB") or
                 Path(__file__).resolve().parent / "_lib" / "libhefv.so")

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_U32 = C.c_uint32

# name -> argtypes (all return int status except where noted)
_SIGS = {
    "hefv_abi_version": [],
    "hefv_ctx_create": [C.POINTER(_P), _U32, _I32, _P, _P, _I32, _P, _P],
    "hefv_ntt_fwd32": [_P, _P, _P, _I64, _I32, _I32, _I32, _P],
    "hefv_ntt_inv32": [_P, _P, _P, _I64, _I32, _I32, _I32, _P],
    "hefv_ntt_fwd64": [_P, _P, _P, _I64, _I32, _I32, _I32, _P],
    "hefv_ntt_inv64": [_P, _P, _P, _I64, _I32, _I32, _I32, _P],
    "hefv_pointwise_mul": [_P, _I32, _P, _P, _P, _I64, _I32, _I32, _P],
    "hefv_fv_setup": [_P, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P],
    "hefv_encode": [_P, _P, _P, _I64, _P],
    "hefv_decode": [_P, _P, _P, _I64, _P],
    "hefv_encode_sparse": [_P, _P, _P, _P, _P, _I64, _P],
    "hefv_plain_to_rns": [_P, _P, _P, _I64, _I32, _I32, _I32, _P],
    "hefv_small_to_rns": [_P, _P, _P, _I64, _I32, _I32, _P],
    "hefv_elementwise": [_P, _I32, _P, _P, _P, _P, _I64, _I64, _I64, _P],
    "hefv_to_montgomery": [_P, _P, _P, _I64, _P],
    "hefv_encrypt": [_P, _P, _P, _P, _P, _P, _P, _I64, _P],
    "hefv_decrypt": [_P, _P, _I32, _P, _P, _P, _P, _I64, _P],
    "hefv_mul_plain": [_P, _P, _P, _P, _I64, _I32, _I32, _P],
    "hefv_rows_mac": [_P, _P, _P, _P, _P, _P, _I64, _P],
    "hefv_automorph": [_P, _P, _I64, _P, _P, _I32, _U32, _I64, _P],
    "hefv_keyswitch": [_P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _I64, _I64, _P],
    "hefv_ks_aux_setup": [_P, _I32],
    "hefv_ks_aux_key": [_P, _P, _P, _P, _P],
    "hefv_ks_aux_key_words": [_P, _P],
    "hefv_keyswitch_aux": [_P, _P, _P, _I64, _P, _U32, _P, _P, _I64, _P, _P, _P, _I64, _P, _P,
                           _I64, _P, _I64, _I64, _P],
    "hefv_keygen_digit": [_P, _P, _P, _I32, _P, _P, _P, _P, _P, _P],
    "hefv_mult_tensor": [_P, _P, _P, _P, _P, _P],
    "hefv_mult_tensor_many": [_P, _P, _I64, _P, _I64, _P, _P, _I64, _P],
    "hefv_accumulate_rows": [_P, _P, _P, _P, _P, _I32, _I32, _P],
    "hefv_add_part0": [_P, _P, _I64, _P, _P, _I64, _P],
    "hefv_rows_mac_indexed": [_P, _P, _P, _P, _P, _P, _P, _I64, _P],
    "hefv_probe_int": [_I32, _I32, _I32, _P, _P],
    "hefv_probe_umma": [_P, _P, _P, _I32, _P],
    "hefv_probe_tmem_shape": [_P, _I32, _P],
    "hefv_probe_umma_lat": [_P, _I32, _I32, _I32, _P],
    "hefv_keyswitch64": [_P, _P, _P, _P, _P, _P, _I64, _P],
    "hefv_to_montgomery64": [_P, _P, _P, _I64, _P],
    "hefv_ks64_aux_setup": [_P, _I32],
    "hefv_ks64_aux_key": [_P, _P, _P, _P, _P, _P],
    "hefv_keyswitch64_aux": [_P, _P, _P, _P, _P, _I64, _P],
    # object-level surface (api.cu) and the C++ layer planner (layer.cu)
    "hefv_ct_alloc": [_P, _I32, _P],
    "hefv_ct_free": [_P, _P],
    "hefv_ct_upload": [_P, _P, _I32, _P, _P],
    "hefv_ct_download": [_P, _P, _I32, _P, _P],
    "hefv_key_upload": [_P, _P, _P, _P, _P],
    "hefv_key_wrap": [_P, _P, _P, _P, _P],
    "hefv_key_free": [_P],
    "hefv_encrypt_slots": [_P, _P, _P, _P, _P, _P, _P, _I64, _P],
    "hefv_decrypt_slots": [_P, _P, _I32, _P, _P, _P, _I64, _P],
    "hefv_add": [_P, _P, _P, _I32, _P, _P],
    "hefv_add_plain": [_P, _P, _I32, _P, _P, _P],
    "hefv_cmult": [_P, _P, _I32, _P, _P, _P],
    "hefv_rotate": [_P, _P, _U32, _P, _P, _P],
    "hefv_mult": [_P, _P, _P, _P, _P, _P],
    "hefv_layer_rows_work_words": [_P, _I32, _I64, _P, _I64, _P],
    "hefv_layer_rows": [_P, _P, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32,
                        _P, _P, _P, _I32, _I64, _P, _I64, _P, _I64, _P],
    "hefv_ks_timing": [_P, _I32],
    "hefv_ks_stats": [_P, _P, _P, _P],
    "hefv_transfer_stats": [_P, _P, _P],
}

EXPORTED = tuple(["hefv_last_error", "hefv_ctx_destroy", "hefv_launch_count"] + list(_SIGS))

# host<->device byte accounting of the Python side (bench.py's e2e fields)
TRAFFIC = {"h2d": 0, "d2h": 0}

_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load(require_cuda: bool = True):
    """Load libhefv.so (once).  Raises NativeError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise NativeError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(_LIB_PATH))
    lib.hefv_last_error.restype = C.c_char_p
    lib.hefv_last_error.argtypes = []
    lib.hefv_ctx_destroy.restype = None
    lib.hefv_ctx_destroy.argtypes = [_P]
    lib.hefv_launch_count.restype = C.c_uint64
    lib.hefv_launch_count.argtypes = []
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = ""):
    if status != 0:
        msg = _lib.hefv_last_error().decode(errors="replace") if _lib else "unknown"
        raise NativeError(f"{what or 'libhefv'} failed ({status}): {msg}")


def call(name: str, *args):
    """Invoke a status-returning ABI function and raise on error."""
    lib = load()
    check(getattr(lib, name)(*args), name)


def launch_count() -> int:
    return int(load().hefv_launch_count())


def to_device(arr):
    """numpy -> CUDA tensor (counted as host-to-device traffic), staged
    through pinned memory and asynchronous on the current stream: a pageable
    copy would make the host wait for every launch queued before it."""
    return to_device_async(arr)


def to_device_async(arr):
    """numpy -> CUDA tensor through pinned memory, asynchronous on the current
    stream (the host keeps enqueueing while the GPU works)."""
    import numpy as np
    import torch

    a = np.ascontiguousarray(arr)
    TRAFFIC["h2d"] += a.nbytes
    return torch.from_numpy(a).pin_memory().to("cuda", non_blocking=True)


def to_host(t):
    """CUDA tensor -> numpy (counted as device-to-host traffic)."""
    TRAFFIC["d2h"] += t.numel() * t.element_size()
    return t.cpu().numpy()


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle():
    import torch

    return torch.cuda.current_stream().cuda_stream


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def require_device():
    if os.environ.get("HEFV_ALLOW_NO_CUDA") != "1" and not cuda_available():
        raise NativeError("no CUDA device visible: the FV backend runs only on the GPU")
