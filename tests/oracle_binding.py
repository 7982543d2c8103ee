"""ctypes binding of oracle/libdgs_oracle.so — the CPU restatement of the
reference algorithm (TEST INFRASTRUCTURE: the checker, never the product)."""
import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent.parent / "oracle" / "libdgs_oracle.so"


class Cam(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("q", C.c_float * 4), ("t", C.c_float * 3)]


class Opts(C.Structure):
    _fields_ = [("trunc", C.c_float), ("near_plane", C.c_float), ("sigma_clamp", C.c_float), ("cov_reg", C.c_float),
                ("stop", C.c_float), ("sh_degree", C.c_int32), ("indicator_enabled", C.c_int32),
                ("grad_skip_eps", C.c_float)]


class Sub(C.Structure):
    _fields_ = [("n", C.c_int32), ("nx", C.c_float * 8), ("ny", C.c_float * 8), ("nz", C.c_float * 8),
                ("d", C.c_float * 8), ("closed", C.c_int32 * 8)]


class Spl(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_coeffs", C.c_int32), ("id", C.c_void_p), ("mu", C.c_void_p),
                ("log_scale", C.c_void_p), ("rotation", C.c_void_p), ("opacity_logit", C.c_void_p),
                ("sh", C.c_void_p)]


class Grads(C.Structure):
    _fields_ = [("d_mu", C.c_void_p), ("d_log_scale", C.c_void_p), ("d_rotation", C.c_void_p),
                ("d_opacity_logit", C.c_void_p), ("d_sh", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(LIB))
        _lib.orc_project.restype = C.c_int64
        _lib.orc_loss.restype = C.c_float
    return _lib


def p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def cam_of(rec):
    c = Cam()
    c.width, c.height = int(rec[0]), int(rec[1])
    c.fx, c.fy, c.cx, c.cy = (float(x) for x in rec[2:6])
    for i in range(4):
        c.q[i] = float(rec[6 + i])
    for i in range(3):
        c.t[i] = float(rec[10 + i])
    return c


def opts(oracle: bool, grad_skip_eps: float = 1e-5):
    o = Opts()
    o.trunc, o.near_plane, o.sigma_clamp, o.cov_reg = 3.0, 0.01, 0.99, 0.3
    o.stop = 0.0 if oracle else 1e-4
    o.sh_degree, o.indicator_enabled, o.grad_skip_eps = -1, 1, grad_skip_eps
    return o


def subspace(planes_k):
    s = Sub()
    s.n = len(planes_k)
    for j, pl in enumerate(planes_k):
        s.nx[j], s.ny[j], s.nz[j], s.d[j] = (float(x) for x in pl[:4])
        s.closed[j] = int(pl[4])
    return s


class Scene:
    """Keeps the numpy arrays alive behind an orc_splats struct."""

    def __init__(self, splats):
        self.s = splats
        self.c = Spl()
        self.c.n, self.c.sh_coeffs = splats.n, splats.sh_coeffs
        self.c.id, self.c.mu, self.c.log_scale = p(splats.id), p(splats.mu), p(splats.log_scale)
        self.c.rotation, self.c.opacity_logit, self.c.sh = p(splats.rotation), p(splats.opacity_logit), p(splats.sh)


def empty_grads(n, shc):
    arrs = dict(d_mu=np.zeros((n, 3), np.float32), d_log_scale=np.zeros((n, 3), np.float32),
                d_rotation=np.zeros((n, 4), np.float32), d_opacity_logit=np.zeros(n, np.float32),
                d_sh=np.zeros((n, shc, 3), np.float32))
    g = Grads(*(p(arrs[k]) for k in ("d_mu", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")))
    return g, arrs
