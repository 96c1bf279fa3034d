"""ctypes binding of libauras_b200.so (the C ABI declared in include/auras_b200.h).

The library is built in-tree (`paper_2509_09560_b200/libauras_b200.so`) by
`__graft_entry__.build()` / `make -C paper_2509_09560_b200/csrc`.  There is no
fallback: importing the engine without the library, or calling it without a
B200, raises `DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError

LIB_PATH = os.environ.get("AURAS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libauras_b200.so")
ABI_VERSION = 4

DT_F32, DT_BF16 = 0, 1
ACT_NONE, ACT_RELU, ACT_MISH, ACT_GELU = 0, 1, 2, 3

vp = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
ip = C.POINTER(C.c_int32)


class ConvOp(C.Structure):
    _fields_ = [
        ("w", vp), ("bias", vp), ("inp", vp), ("out", vp), ("gn_gamma", vp), ("gn_beta", vp),
        ("res", vp), ("res_f32", vp), ("out_f32", vp),
        ("M", i32), ("Cin", i32), ("Kp", i32),
        ("H", i32), ("W", i32), ("in_pitch", i32), ("in_coff", i32),
        ("kh", i32), ("kw", i32), ("stride", i32), ("pad_h", i32), ("pad_w", i32),
        ("Ho", i32), ("Wo", i32), ("out_pitch", i32), ("out_coff", i32),
        ("res_pitch", i32), ("res_coff", i32),
        ("groups", i32), ("act", i32), ("res_before_act", i32), ("film_off", i32),
        ("out_stuff", i32), ("pool_out", i32), ("splits", i32), ("cta_target", i32), ("reserved", i32 * 2),
    ]


class LinearOp(C.Structure):
    _fields_ = [("w", vp), ("bias", vp), ("M", i32), ("K", i32), ("mish_in", i32), ("ldw", i32)]


class DptGemm(C.Structure):
    _fields_ = [("act", vp), ("act_rows", i32), ("K", i32), ("w", vp), ("N", i32), ("bias", vp), ("res", vp),
                ("ldr", i32), ("out", vp), ("ldo", i32), ("out_f32", vp), ("ldf", i32), ("act_fn", i32),
                ("ln_src", vp), ("ln_g", vp), ("ln_b", vp), ("ksplit", i32), ("fuse_update", i32), ("a_from_lanes", i32)]


class DptOp(C.Structure):
    _fields_ = [("type", i32), ("gemm", i32), ("inp", vp), ("out", vp), ("g", vp), ("b", vp), ("k", vp), ("v", vp),
                ("ldi", i32), ("ldo", i32), ("ldk", i32), ("ldv", i32), ("nk", i32), ("mask_off", i32),
                ("heads", i32), ("dh", i32), ("qrows", i32), ("krows", i32), ("k2", vp), ("v2", vp),
                ("k2rows", i32), ("gather", i32)]


class Sched(C.Structure):
    _fields_ = [("timestep", vp), ("sqrt_ab", vp), ("sqrt_1mab", vp), ("c_x0", vp), ("c_xt", vp),
                ("c_eps", vp), ("sigma", vp), ("n_steps", i32), ("clip_sample", i32), ("ddpm", i32),
                ("reserved", i32)]


_SIGNATURES = {
    "auras_last_error": (C.c_char_p, []),
    "auras_abi_version": (C.c_int, []),
    "auras_device_ok": (C.c_int, [C.c_int]),
    "auras_ring_commit": (C.c_int, [vp, vp, C.c_int, i64, i64, vp]),
    "auras_ring_fetch": (C.c_int, [vp, vp, C.c_int, i64, vp, vp, i64, vp]),
    "auras_ring_commit_sys": (C.c_int, [vp, vp, C.c_int, i64, i64, vp]),
    "auras_enable_peer": (C.c_int, [C.c_int, C.c_int]),
    "auras_peer_copy": (C.c_int, [vp, i64, vp, i64, i64, i64, vp]),
    "auras_ring_write": (C.c_int, [vp, i64, C.c_int, vp, i64, vp]),
    "auras_toy_ingest": (C.c_int, [vp, C.c_int, C.POINTER(f64), vp, C.POINTER(f64), vp]),
    "auras_toy_publish": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int, i64, i64, vp]),
    "auras_toy_generate": (C.c_int, [vp, ip, ip, C.c_int, f64, vp, vp, vp]),
    "auras_toy_finish": (C.c_int, [vp, C.c_int, f64, vp, vp]),
    "auras_ar_generate": (C.c_int, [vp, C.c_int, ip, ip, ip, C.c_int, vp, vp, f64, vp]),
    "auras_ar_finish": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "auras_ring_copy_slot": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp]),
    "auras_conv_ln": (C.c_int, [C.POINTER(ConvOp), C.c_int, C.c_int, vp, vp, vp, C.c_int, C.c_float, vp, i64, vp]),
    "auras_conv_scratch_floats": (i64, [C.POINTER(ConvOp), C.c_int, C.c_int]),
    "auras_dpt_prep": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, vp, i64, C.c_int, vp,
                                 C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp]),
    "auras_dpt_cond": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp]),
    "auras_dpt_kv_gather": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp]),
    "auras_attention": (C.c_int, [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_int, vp]),
    "auras_dpt_update": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(Sched), vp]),
    "auras_vit_tokens": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
    "auras_layernorm": (C.c_int, [vp, i64, vp, i64, C.c_int, vp, vp, C.c_int, C.c_int, C.c_float, vp]),
    "auras_vit_attention": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
    "auras_tf_param_count": (i64, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "auras_tf_forward": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int,
                                   vp, vp, vp, vp, vp]),
    "auras_tf_logits": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp]),
    "auras_unet_plan_create": (vp, [C.POINTER(ConvOp), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    vp, vp, C.c_int, i64, i64, vp, vp, C.c_int, C.POINTER(Sched),
                                    vp, C.c_int]),
    "auras_unet_plan_destroy": (None, [vp]),
    "auras_unet_generate": (C.c_int, [vp, C.c_int, ip, ip, ip, ip, C.c_int, C.c_int, vp, vp, vp,
                                      C.c_int, vp]),
    "auras_unet_mega_trace": (C.c_int, [vp, C.c_int, vp, vp, C.c_int]),
    "auras_unet_kernel_for": (C.c_int, [vp, C.c_int]),
    "auras_unet_check": (C.c_int, [vp]),
    "auras_ring_stress": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, vp]),
    "auras_host_mapped_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp), C.POINTER(vp)]),
    "auras_host_mapped_free": (C.c_int, [vp]),
    "auras_dpt_persist_build": (C.c_int, [C.POINTER(DptGemm), C.c_int, C.POINTER(DptOp), C.c_int, C.c_int,
                                          C.POINTER(vp)]),
    "auras_dpt_persist_run": (C.c_int, [vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(Sched), vp]),
    "auras_dpt_persist_free": (None, [vp]),
    "auras_dpt_persist_trace": (C.c_int, [vp, vp, C.c_int]),
    "auras_dpt_xfold": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp,
                                  C.c_int, vp]),
    "auras_unet_launches_per_iter": (C.c_int, [vp]),
    "auras_conv": (C.c_int, [C.POINTER(ConvOp), C.c_int, C.c_int, vp, C.c_int, vp, i64, vp]),
    "auras_linear": (C.c_int, [C.POINTER(LinearOp), C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, vp]),
    "auras_image_to_nhwc": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int,
                                      vp]),
    "auras_maxpool3s2": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp]),
    "auras_dp_assemble_cond": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         vp, i64, vp]),
    "auras_sinusoidal": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "auras_dp_copy_rows": (C.c_int, [vp, vp, i64, vp]),
    "auras_dp_finish": (C.c_int, [vp, C.c_int, ip, ip, C.c_int, C.c_int, C.c_int, vp, vp]),
}

_lock = threading.Lock()
_lib = None
_checked_devices = set()


def exported_symbols():
    return sorted(_SIGNATURES)


def load(require_device: bool = True):
    """Load the native library (once).  Raises DeviceError when it is missing,
    stale, or -- with require_device -- when no sm_100 device is present."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.auras_abi_version() != ABI_VERSION:
                raise DeviceError("libauras_b200.so ABI mismatch; rebuild it")
            _lib = lib
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("the B200 engine needs a CUDA device; none is visible")
        dev = torch.cuda.current_device()
        if dev not in _checked_devices:        # cudaGetDeviceProperties costs milliseconds: once per device
            if not _lib.auras_device_ok(dev):
                raise DeviceError(f"device {torch.cuda.get_device_name(dev)} is not sm_100 (B200)")
            _checked_devices.add(dev)
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.auras_last_error().decode() if _lib is not None else "?"
        raise DeviceError(f"{what}: {msg} (code {rc})")


def ptr(t) -> int:
    """Device (or host) address of a torch tensor, or 0 for None."""
    return 0 if t is None else t.data_ptr()


def int_array(values):
    arr = (C.c_int32 * max(1, len(values)))(*values)
    return arr


def stream_handle(stream) -> int:
    return stream.cuda_stream
