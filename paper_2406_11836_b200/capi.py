"""ctypes binding of libdgs_b200.so (include/dgs_capi.h).

The library is the product: sm_100a kernels + C-ABI + host C++.  There is no
Python or CPU fallback — if the shared object is missing or a call fails, an
exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
# DGS_LIB: an alternative build of the same library (compile-time variants in scripts/)
LIB_PATH = Path(os.environ["DGS_LIB"]) if os.environ.get("DGS_LIB") else _HERE / "libdgs_b200.so"

DGS_OK = 0
_ERRORS = {1: ValueError, 2: RuntimeError, 3: ArithmeticError, 4: RuntimeError, 5: RuntimeError}


class DgsCudaError(RuntimeError):
    pass


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("q_wc", C.c_float * 4), ("t_wc", C.c_float * 3)]

    def record(self) -> np.ndarray:
        """[w, h, fx, fy, cx, cy, qw, qx, qy, qz, tx, ty, tz] (oracle/ref_dump camera record)."""
        return np.array([self.width, self.height, self.fx, self.fy, self.cx, self.cy, *self.q_wc, *self.t_wc],
                        dtype=np.float32)

    @classmethod
    def from_record(cls, r) -> "Camera":
        r = np.asarray(r, dtype=np.float32)
        c = cls()
        c.width, c.height = int(r[0]), int(r[1])
        c.fx, c.fy, c.cx, c.cy = (float(x) for x in r[2:6])
        for i in range(4):
            c.q_wc[i] = float(r[6 + i])
        for i in range(3):
            c.t_wc[i] = float(r[10 + i])
        return c


class RenderOptionsC(C.Structure):
    _fields_ = [("truncation_radius", C.c_double), ("near_plane", C.c_double), ("sigma_clamp", C.c_double),
                ("cov2d_regularization", C.c_double), ("stop_threshold", C.c_double), ("sh_degree", C.c_int32),
                ("indicator_enabled", C.c_int32), ("camera_z_order", C.c_int32), ("grad_skip_eps", C.c_double)]


class TrainConfigC(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("batch_size", C.c_int32), ("kd_depth", C.c_int32),
                ("lambda_ssim", C.c_double), ("lr_position_start", C.c_double), ("lr_position_end", C.c_double),
                ("lr_sh_dc", C.c_double), ("lr_sh_rest", C.c_double), ("lr_opacity", C.c_double),
                ("lr_scale", C.c_double), ("lr_rotation", C.c_double), ("adam_beta1", C.c_double),
                ("adam_beta2", C.c_double), ("adam_eps", C.c_double), ("grad_sync", C.c_int32),
                ("deterministic", C.c_int32)]


class Plane(C.Structure):
    _fields_ = [("n", C.c_float * 3), ("d", C.c_float), ("closed", C.c_int32)]


class SplatsC(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_coeffs", C.c_int32), ("id", C.POINTER(C.c_uint64)),
                ("mu", C.POINTER(C.c_float)), ("log_scale", C.POINTER(C.c_float)),
                ("rotation", C.POINTER(C.c_float)), ("opacity_logit", C.POINTER(C.c_float)),
                ("sh", C.POINTER(C.c_float))]


XFER_SEND = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
XFER_RECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
XFER_FLUSH = C.CFUNCTYPE(C.c_int, C.c_void_p)
XFER_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_uint64)


class HostTransportC(C.Structure):
    """dgs_host_transport: test transport of the multi-rank step."""
    _fields_ = [("user", C.c_void_p), ("send", XFER_SEND), ("recv", XFER_RECV), ("flush", XFER_FLUSH),
                ("allreduce_sum_f64", XFER_ALLREDUCE)]


class StepResult(C.Structure):
    _fields_ = [("loss", C.c_double), ("psnr", C.c_double), ("comm_bytes", C.c_uint64), ("nccl_bytes", C.c_uint64),
                ("pairs", C.c_uint64), ("evals_fwd", C.c_uint64), ("contribs_fwd", C.c_uint64),
                ("evals_bwd", C.c_uint64), ("contribs_bwd", C.c_uint64), ("overflow_pixels", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("subrounds_bwd", C.c_uint64),
                ("small_subrounds_bwd", C.c_uint64), ("tiles_work_fwd", C.c_uint64),
                ("replay_tiles_bwd", C.c_uint64), ("visible", C.c_uint64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = C.c_void_p
_SIGS = {
    "dgs_last_error": (C.c_char_p, []),
    "dgs_version": (C.c_int, []),
    "dgs_default_render_options": (None, [C.POINTER(RenderOptionsC)]),
    "dgs_oracle_render_options": (None, [C.POINTER(RenderOptionsC)]),
    "dgs_default_train_config": (None, [C.POINTER(TrainConfigC)]),
    "dgs_position_lr": (C.c_double, [C.POINTER(TrainConfigC), C.c_uint64]),
    "dgs_build_kdtree": (C.c_int, [_P, C.c_int64, C.c_int32, C.POINTER(Plane)]),
    "dgs_assign_subsets": (C.c_int, [C.POINTER(Plane), C.c_int32, C.c_int32, _P, _P, C.c_int64, C.c_double, _P]),
    "dgs_synth_splats": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.POINTER(SplatsC)]),
    "dgs_ring_camera": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                  C.POINTER(Camera)]),
    "dgs_perturb_splats": (C.c_int, [C.POINTER(SplatsC), C.c_uint64]),
    "dgs_nccl_unique_id": (C.c_int, [_P]),
    "dgs_nccl_selftest": (C.c_int, [C.c_int32]),
    "dgs_ctx_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _P, C.POINTER(_P)]),
    "dgs_ctx_create_host_transport": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(HostTransportC),
                                              C.POINTER(_P)]),
    "dgs_ctx_destroy": (C.c_int, [_P]),
    "dgs_set_table": (C.c_int, [_P, C.POINTER(Plane), C.c_int32, C.c_int32]),
    "dgs_set_options": (C.c_int, [_P, C.POINTER(RenderOptionsC), C.POINTER(TrainConfigC)]),
    "dgs_subset_load": (C.c_int, [_P, C.c_int32, C.POINTER(SplatsC), C.POINTER(SplatsC), C.POINTER(SplatsC),
                                  C.c_uint64, C.c_uint64]),
    "dgs_repartition": (C.c_int, [_P, C.c_int32, C.c_double, C.c_int64, C.c_uint64, C.POINTER(Plane)]),
    "dgs_subset_ids": (C.c_int, [_P, C.c_int32, _P]),
    "dgs_init_from_pointcloud": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                         C.POINTER(SplatsC)]),
    "dgs_save_splats_ply": (C.c_int, [C.POINTER(SplatsC), C.c_char_p, C.c_int32]),
    "dgs_load_splats_ply": (C.c_int, [C.c_char_p, C.POINTER(SplatsC), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "dgs_subset_store": (C.c_int, [_P, C.c_int32, C.POINTER(SplatsC), C.POINTER(SplatsC), C.POINTER(SplatsC),
                                   C.POINTER(C.c_uint64)]),
    "dgs_subset_size": (C.c_int64, [_P, C.c_int32]),
    "dgs_set_epoch": (C.c_int, [_P, C.c_uint64]),
    "dgs_render_partial": (C.c_int, [_P, C.c_int32, C.POINTER(Camera), _P, C.c_int32, _P, _P]),
    "dgs_dump_bins": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "dgs_dump_records": (C.c_int, [_P, C.c_int32, _P, _P]),
    "dgs_pixel_orders": (C.c_int, [_P, C.POINTER(Camera), _P, _P]),
    "dgs_merge": (C.c_int, [_P, C.POINTER(Camera), _P, _P, _P, _P]),
    "dgs_loss": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, C.c_double, C.c_double, _P, C.POINTER(C.c_double), _P]),
    "dgs_merge_backward": (C.c_int, [_P, C.POINTER(Camera), _P, _P, _P, _P]),
    "dgs_merge_ordered": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "dgs_merge_backward_ordered": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P,
                                             _P, _P]),
    "dgs_render_partial_backward": (C.c_int, [_P, C.c_int32, C.POINTER(Camera), _P, C.POINTER(SplatsC)]),
    "dgs_dump_pixel_grads": (C.c_int, [_P, C.c_int32, _P]),
    "dgs_adam_apply": (C.c_int, [_P, C.c_int32, C.POINTER(SplatsC)]),
    "dgs_train_step": (C.c_int, [_P, C.c_int32, C.POINTER(Camera), _P, C.c_int32, _P, C.POINTER(StepResult)]),
    "dgs_upload_targets": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, C.POINTER(_P)]),
    "dgs_render": (C.c_int, [_P, C.POINTER(Camera), _P, _P, _P]),
    "dgs_set_profiling": (C.c_int, [_P, C.c_int32]),
    "dgs_set_collect_stats": (C.c_int, [_P, C.c_int32]),
    "dgs_stage_times": (C.c_int, [_P, _P, _P]),
    "dgs_set_backward_records": (C.c_int, [_P, C.c_int32]),
    "dgs_set_virtual_slices": (C.c_int, [_P, C.c_int32]),
    "dgs_slice_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _P]),
    "dgs_subset_owner": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32]),
    "dgs_dump_grad_maps": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    "dgs_stream": (_P, [_P]),
    "dgs_sync": (C.c_int, [_P]),
    "dgs_set_graph_mode": (C.c_int, [_P, C.c_int32]),
    "dgs_state_save": (C.c_int, [_P]),
    "dgs_state_restore": (C.c_int, [_P]),
}

STAGES = ("preprocess", "binning", "blend_fwd", "merge", "loss", "merge_bwd", "blend_bwd", "project_bwd", "adam",
          "exchange")

_lib = None


def lib() -> C.CDLL:
    """Load libdgs_b200.so (built by __graft_entry__.build()).  Fails loudly."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("DGS_LIB") and not hasattr(L, name):
                continue  # an older build under A/B timing (DGS_LIB): entry points it lacks stay unbound
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != DGS_OK:
        msg = lib().dgs_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(f"dgs error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C-ABI must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def declared_symbols() -> list[str]:
    """Every function declared in include/dgs_capi.h."""
    import re
    hdr = (_HERE.parent / "include" / "dgs_capi.h").read_text()
    return sorted(set(re.findall(r"\b(dgs_[a-z0-9_]+)\s*\(", hdr)))
