"""ctypes binding of the C ABI (include/tsunami_b200.h).

The library is built in-tree (``python -m paper_2408_07609_b200.build``) and
loaded from this package directory only.  There is no CPU fallback: if the
library is missing or no CUDA device is usable, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import weakref

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSUNAMI_B200_LIB") or os.path.join(HERE, "libtsunami_b200.so")

TS_OK, TS_ERR_NUMERICS, TS_ERR_CUDA, TS_ERR_INVALID = 0, 1, 2, 3
ABI_VERSION = 2

FIELDS = {"eta_old": 0, "eta_new": 1, "m_old": 2, "m_new": 3, "n_old": 4, "n_new": 5,
          "h_ext": 6, "max_eta": 7, "max_speed": 8, "max_inundation": 9}
PHASES = {"mass": 0, "restrict": 1, "halo-eta": 2, "momentum": 3, "edges": 4, "prolong": 5,
          "halo-flux": 6, "output": 7, "swap": 8}

c_int32, c_int64, c_double, c_void_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
PD = ctypes.POINTER(ctypes.c_double)


class BlockDesc(ctypes.Structure):
    _fields_ = [("block_id", c_int64), ("ni", c_int32), ("nj", c_int32), ("owner", c_int32),
                ("level", c_int32), ("dx", c_double), ("manning", c_double), ("h_ext", PD),
                ("nman_ext", PD), ("eta0", PD), ("h_profile", PD), ("h_axis", c_int32), ("pad_", c_int32)]


class HaloEntryC(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("sender", "receiver", "side", "send_lo", "send_hi",
                                       "recv_lo", "recv_hi")]


class EtaSegmentC(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("parent", "child", "side", "child_lo", "child_hi",
                                       "ring_start", "parent_line", "parent_lo", "parent_hi")]


class FluxSegmentC(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("parent", "child", "side", "child_lo", "child_hi",
                                       "child_face_line", "parent_face_line", "parent_lo",
                                       "parent_hi")]


class EdgeC(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("block", "side", "kind", "lo", "hi")]


class Desc(ctypes.Structure):
    _fields_ = [("abi_version", c_int32), ("n_blocks", c_int32), ("blocks", ctypes.POINTER(BlockDesc)),
                ("dt", c_double), ("gravity", c_double), ("wet_threshold", c_double),
                ("n_halo", c_int32), ("halo", ctypes.POINTER(HaloEntryC)),
                ("n_restrict", c_int32), ("restrict_segs", ctypes.POINTER(EtaSegmentC)),
                ("n_prolong", c_int32), ("prolong_segs", ctypes.POINTER(FluxSegmentC)),
                ("n_edges", c_int32), ("edges", ctypes.POINTER(EdgeC)),
                ("rank", c_int32), ("n_ranks", c_int32), ("device", c_int32),
                ("tile_rows", c_int32)]


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_LIB = None


def lib():
    """Load the in-tree CUDA library (fails loudly; never falls back)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2408_07609_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    L.ts_last_error.restype = ctypes.c_char_p
    L.ts_abi_version.restype = c_int32
    L.ts_create.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(c_void_p)]
    L.ts_run.argtypes = [c_void_p, c_int64]
    L.ts_phase.argtypes = [c_void_p, c_int32]
    L.ts_get_field.argtypes = [c_void_p, c_int32, c_int32, c_void_p, c_int64]
    L.ts_set_field.argtypes = [c_void_p, c_int32, c_int32, c_void_p, c_int64]
    L.ts_set_initial_eta.argtypes = [c_void_p, c_int32, c_void_p, c_int64]
    L.ts_host_alloc.argtypes = [c_int64]
    L.ts_host_alloc.restype = c_void_p
    L.ts_host_free.argtypes = [c_void_p]
    L.ts_host_free.restype = None
    L.ts_error_info.argtypes = [c_void_p] + [c_void_p] * 4
    L.ts_timings.argtypes = [c_void_p, c_void_p, c_void_p]
    L.ts_steps_done.argtypes = [c_void_p]
    L.ts_steps_done.restype = c_int64
    L.ts_device_bytes.argtypes = [c_void_p]
    L.ts_device_bytes.restype = c_int64
    L.ts_launches_per_step.argtypes = [c_void_p]
    L.ts_launches_per_step.restype = c_int32
    L.ts_set_timing.argtypes = [c_void_p, c_int32]
    L.ts_trace_step.argtypes = [c_void_p, c_void_p, c_void_p, c_int32, c_void_p]
    L.ts_device_barrier.argtypes = [c_void_p]
    L.ts_kernel_seconds.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
    L.ts_stream.argtypes = [c_void_p, ctypes.POINTER(c_void_p)]
    L.ts_destroy.argtypes = [c_void_p]
    L.ts_destroy.restype = None
    L.ts_ipc_export.argtypes = [c_void_p, c_void_p, c_int64]
    L.ts_ipc_import.argtypes = [c_void_p, c_int32, c_void_p, c_int64]
    L.ts_cbrt_host.argtypes = [c_void_p, c_void_p, c_int64]
    L.ts_cbrt_host.restype = None
    L.ts_cbrt_device.argtypes = [c_int32, c_void_p, c_void_p, c_int64]
    L.ts_reset.argtypes = [c_void_p]
    L.ts_upload_inputs.argtypes = [c_void_p, c_int32, c_void_p, c_void_p, c_void_p]
    L.ts_download_fields.argtypes = [c_void_p, c_int32, c_void_p, c_int32, c_void_p, c_void_p]
    L.ts_upload_profiles.argtypes = [c_void_p, c_int32, c_void_p, c_void_p, c_void_p]
    if L.ts_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI {L.ts_abi_version()} != {ABI_VERSION}")
    _LIB = L
    return L


EXPORTED = ("ts_last_error", "ts_abi_version", "ts_create", "ts_run", "ts_phase", "ts_get_field",
            "ts_set_field", "ts_error_info", "ts_timings", "ts_steps_done", "ts_device_bytes",
            "ts_launches_per_step", "ts_set_timing", "ts_trace_step", "ts_device_barrier", "ts_kernel_seconds", "ts_stream", "ts_destroy",
            "ts_ipc_export", "ts_ipc_import", "ts_cbrt_host", "ts_cbrt_device", "ts_set_initial_eta",
            "ts_host_alloc", "ts_host_free", "ts_reset", "ts_upload_inputs", "ts_download_fields", "ts_upload_profiles")


def pinned_empty(shape) -> np.ndarray:
    """A float64 array in page-locked host memory (ts_host_alloc), freed when
    the array is garbage collected."""
    n = int(np.prod(shape))
    p = lib().ts_host_alloc(max(1, n) * 8)
    if not p:
        raise MemoryError(f"ts_host_alloc of {n * 8} bytes failed")
    buf = (ctypes.c_double * max(1, n)).from_address(p)
    arr = np.frombuffer(buf, dtype=np.float64, count=n).reshape(shape)
    weakref.finalize(buf, lib().ts_host_free, p)
    return arr


def check(rc: int):
    if rc != TS_OK:
        raise NativeError(rc, lib().ts_last_error().decode())


def cbrt_host(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(a)
    lib().ts_cbrt_host(a.ctypes.data, out.ctypes.data, a.size)
    return out


def cbrt_device(x, device: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(a)
    check(lib().ts_cbrt_device(device, a.ctypes.data, out.ctypes.data, a.size))
    return out
