"""ctypes binding of the C ABI in include/hcnn_b200.h.

This is the only place Python touches the CUDA engine.  There is no CPU
fallback: if ``libhcnn_b200.so`` is missing or no CUDA device is visible,
every entry point raises ``NativeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import (
    BasisError,
    DomainError,
    HcnnError,
    KeyError_,
    LevelError,
    NativeError,
    ParameterError,
    ScaleError,
)

LIB_NAME = "libhcnn_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

_VP = ctypes.c_void_p
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_INT = ctypes.c_int
_SZ = ctypes.c_size_t
_PU64 = ctypes.POINTER(ctypes.c_uint64)
_PU32 = ctypes.POINTER(ctypes.c_uint32)

# name -> (restype, argtypes); keep in sync with include/hcnn_b200.h
SIGNATURES = {
    "hcnn_last_error": (ctypes.c_char_p, []),
    "hcnn_abi_version": (_INT, []),
    "hcnn_ctx_create": (_INT, [ctypes.POINTER(_VP), _INT, _U32, _PU64, _U32, _PU64, _U32]),
    "hcnn_ctx_destroy": (None, [_VP]),
    "hcnn_ctx_psi": (_INT, [_VP, _U32, _PU64]),
    "hcnn_ntt_forward": (_INT, [_VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_ntt_inverse": (_INT, [_VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_poly_add": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _U32, _INT, _VP]),
    "hcnn_poly_sub": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _U32, _INT, _VP]),
    "hcnn_poly_neg": (_INT, [_VP, _VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_poly_mul": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _U32, _INT, _VP]),
    "hcnn_poly_mul_mont": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _U32, _INT, _VP]),
    "hcnn_poly_mac_mont": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _U32, _INT, _VP]),
    "hcnn_to_mont": (_INT, [_VP, _VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_from_mont": (_INT, [_VP, _VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_scalar_mul": (_INT, [_VP, _VP, _VP, _PU64, _U32, _U32, _U32, _VP]),
    "hcnn_scalar_add": (_INT, [_VP, _VP, _VP, _PU64, _U32, _U32, _U32, _VP]),
    "hcnn_from_signed": (_INT, [_VP, _VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_ntt_from_signed": (_INT, [_VP, _VP, _VP, _U32, _U32, _INT, _VP]),
    "hcnn_from_signed_mont": (_INT, [_VP, _VP, _VP, _U32, _U32, _U32, _VP]),
    "hcnn_automorphism": (_INT, [_VP, _VP, _VP, _U64, _INT, _U32, _U32, _U32, _VP]),
    "hcnn_base_convert": (_INT, [_VP, _VP, _VP, _PU32, _U32, _PU32, _U32, _U32, _VP]),
    "hcnn_ks_workspace_bytes": (_SZ, [_VP, _U32]),
    "hcnn_keyswitch": (_INT, [_VP, _VP, _VP, _VP, _U32, _VP, _VP, _VP, _VP]),
    "hcnn_hmult": (_INT, [_VP, _VP, _VP, _VP, _U32, _VP, _VP, _VP, _VP]),
    "hcnn_rotate_hoisted": (_INT, [_VP, ctypes.POINTER(_VP), _VP, _U32, _U32, _PU64,
                                   ctypes.POINTER(_VP), ctypes.POINTER(_VP), _VP, _VP]),
    "hcnn_ks_workspace_bytes_batch": (_SZ, [_VP, _U32, _U32]),
    "hcnn_ks_workspace_bytes_rot": (_SZ, [_VP, _U32, _U32, _U32]),
    "hcnn_hmult_batch": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _VP, _VP, _VP, _VP]),
    "hcnn_rotate_hoisted_batch": (_INT, [_VP, ctypes.POINTER(_VP), _VP, _U32, _U32, _U32, _PU64,
                                         ctypes.POINTER(_VP), ctypes.POINTER(_VP), _PU32, _VP, _VP]),
    "hcnn_mac_terms_multi": (_INT, [_VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP), ctypes.POINTER(_VP), _U32, _U32,
                                    _U32, _INT, _VP]),
    "hcnn_mac_terms_multi_packed": (_INT, [_VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP), ctypes.POINTER(_VP),
                                           ctypes.POINTER(ctypes.c_ubyte), _U32, _U32, _U32, _INT, _VP]),
    "hcnn_mac_terms_multi_images": (_INT, [_VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP), ctypes.POINTER(_VP),
                                           ctypes.POINTER(ctypes.c_ubyte), _U32, _U32, _U32, _U32, _INT, _VP]),
    "hcnn_pack_masks": (_INT, [_VP, _VP, _VP, _U32, _U32, _VP]),
    "hcnn_unpack_mask": (_INT, [_VP, _VP, _VP, _U32, _VP]),
    "hcnn_mac_terms_batch": (_INT, [_VP, _VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP), _U32, _U32, _U32, _INT,
                                    _VP]),
    "hcnn_rotate_hoisted_ext_batch": (_INT, [_VP, ctypes.POINTER(_VP), _VP, _U32, _U32, _U32, _PU64,
                                             ctypes.POINTER(_VP), ctypes.POINTER(_VP), _PU32, _VP, _VP]),
    "hcnn_mac_terms_ext_batch": (_INT, [_VP, _VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP), _U32, _U32, _U32,
                                        _INT, _VP]),
    "hcnn_moddown_batch": (_INT, [_VP, _VP, _VP, _U32, _U32, _VP, _VP]),
    "hcnn_moddown_rescale_batch": (_INT, [_VP, _VP, _VP, _U32, _U32, _VP, _VP]),
    "hcnn_hmult_rescale_workspace_bytes": (ctypes.c_size_t, [_VP, _U32, _U32]),
    "hcnn_hmult_rescale_batch": (_INT, [_VP, _VP, _VP, _VP, _U32, _U32, _VP, _VP, _VP, _VP]),
    "hcnn_rescale_workspace_bytes": (_SZ, [_VP, _U32]),
    "hcnn_rescale": (_INT, [_VP, _VP, _VP, _U32, _U32, _VP, _VP]),
    "hcnn_scalar_mac": (_INT, [_VP, _VP, ctypes.POINTER(_VP), ctypes.POINTER(_U32), _PU64, _U32, _U32, _U32, _INT,
                               _PU64, _VP]),
    "hcnn_mac_terms": (_INT, [_VP, _VP, ctypes.POINTER(_VP), ctypes.POINTER(_VP), _U32, _U32, _INT, _VP]),
    "hcnn_kernel_launches": (ctypes.c_ulonglong, []),
    "hcnn_profile_enable": (None, [_INT]),
    "hcnn_ntt_butterfly_peak": (_INT, [_INT, _INT, ctypes.POINTER(ctypes.c_double)]),
    "hcnn_ntt_limb_counts": (None, [ctypes.POINTER(ctypes.c_ulonglong), _INT]),
    "hcnn_ks_counters": (None, [ctypes.POINTER(ctypes.c_ulonglong), _INT]),
    "hcnn_set_option": (_INT, [ctypes.c_char_p, ctypes.c_longlong]),
    "hcnn_profile_read": (_INT, [ctypes.c_char_p, _SZ, _INT]),
}

_STATUS = {
    1: ParameterError,
    2: DomainError,
    3: BasisError,
    4: LevelError,
    5: ScaleError,
    6: KeyError_,
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load the engine (once).  Fails loudly: there is no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("HCNN_B200_LIB", str(LIB_PATH))
        if not os.path.exists(path):
            raise NativeError(
                f"CUDA engine {path} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        # tuning knobs from the environment: HCNN_OPTIONS="ntt_occupancy=1,merge_moddown=0"
        for item in filter(None, os.environ.get("HCNN_OPTIONS", "").split(",")):
            key, _, val = item.partition("=")
            if lib.hcnn_set_option(key.strip().encode(), int(val or 1)) != 0:
                raise NativeError(f"unknown HCNN_OPTIONS entry {item!r}")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load().hcnn_last_error() or b"").decode(errors="replace")
    cls = _STATUS.get(rc, NativeError)
    raise cls(f"hcnn-b200: {msg} (status {rc})")


def kernel_launches() -> int:
    return int(load().hcnn_kernel_launches())


def ntt_butterfly_peak(fast: bool, device: int = 0) -> float:
    """Measured butterflies/s of the NTT's register network (integer-pipe ceiling)."""
    out = ctypes.c_double(0.0)
    check(load().hcnn_ntt_butterfly_peak(int(device), int(fast), ctypes.byref(out)))
    return float(out.value)


def ntt_limb_counts(reset: bool = True) -> dict:
    """Limbs transformed since the last reset: fwd/inv x (q < 2^47 fast path, full)."""
    buf = (ctypes.c_ulonglong * 4)()
    load().hcnn_ntt_limb_counts(buf, 1 if reset else 0)
    return {"fwd_fast": buf[0], "fwd_full": buf[1], "inv_fast": buf[2], "inv_full": buf[3]}


def ks_counters(reset: bool = True) -> dict:
    """Key switches since the last reset with their minimal HBM bytes and limb-NTT counts."""
    buf = (ctypes.c_ulonglong * 4)()
    load().hcnn_ks_counters(buf, 1 if reset else 0)
    return {"keyswitches": buf[0], "min_bytes": buf[1], "fwd_limbs": buf[2], "inv_limbs": buf[3]}


def set_option(name: str, value: int) -> None:
    check(load().hcnn_set_option(name.encode(), int(value)))


def profile_enable(on: bool) -> None:
    load().hcnn_profile_enable(1 if on else 0)


def profile_read(reset: bool = True) -> dict:
    """{kernel: {"launches", "ms", "bytes", "kernels"}} accumulated since the last reset."""
    import json
    lib = load()
    n = lib.hcnn_profile_read(None, 0, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib.hcnn_profile_read(buf, n + 1, 1 if reset else 0)
    raw = json.loads(buf.value.decode())
    return {k: {"launches": int(v[0]), "ms": v[1], "bytes": v[2], "kernels": int(v[3])} for k, v in raw.items()}


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def u64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_uint64 * len(vals))(*vals)


def u32_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_uint32 * len(vals))(*vals)


__all__ = ["load", "check", "exported_symbols", "u64_array", "u32_array", "LIB_PATH", "HcnnError"]
