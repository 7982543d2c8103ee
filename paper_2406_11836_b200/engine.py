"""Host-side mirror of the reference's public API for the hot path.

Names, argument meaning and error behaviour follow /root/reference/proj/include/dgs
(`build_kdtree`/`assign_subsets` partition.hpp:160-251, `partial_render`
engine.hpp:44-52, `compute_pixel_orders` engine.hpp:108-131, `merge`
engine.hpp:152-182, `merge_backward` engine.hpp:195-234, `loss` loss.hpp:153-177,
`partial_render_backward` engine.hpp:74-88, `adam_apply` optim.hpp:104-126,
`Manager::train_step` manager.hpp:313-386).  Everything here is plumbing over
the C-ABI of libdgs_b200.so; all compute runs in the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import Camera, Plane, StepResult, check, fptr, lib, ptr


# ---------------------------------------------------------------------------
# Options
# ---------------------------------------------------------------------------
def render_options(oracle: bool = False, **overrides) -> capi.RenderOptionsC:
    o = capi.RenderOptionsC()
    (lib().dgs_oracle_render_options if oracle else lib().dgs_default_render_options)(C.byref(o))
    for k, v in overrides.items():
        setattr(o, k, v)
    return o


def train_config(**overrides) -> capi.TrainConfigC:
    c = capi.TrainConfigC()
    lib().dgs_default_train_config(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def position_lr(cfg: capi.TrainConfigC, step: int) -> float:
    return lib().dgs_position_lr(C.byref(cfg), step)


# ---------------------------------------------------------------------------
# Splats (host SoA mirror of std::vector<Splat<float>>)
# ---------------------------------------------------------------------------
@dataclass
class Splats:
    id: np.ndarray
    mu: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray
    opacity_logit: np.ndarray
    sh: np.ndarray
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n(self) -> int:
        return int(self.id.shape[0])

    @property
    def sh_coeffs(self) -> int:
        return int(self.sh.shape[1])

    @classmethod
    def empty(cls, n: int, sh_coeffs: int = 16) -> "Splats":
        return cls(np.zeros(n, np.uint64), np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32),
                   np.zeros((n, 4), np.float32), np.zeros(n, np.float32), np.zeros((n, sh_coeffs, 3), np.float32))

    @classmethod
    def load_npy(cls, d, prefix: str = "scene_") -> "Splats":
        from pathlib import Path
        d = Path(d)
        return cls(np.load(d / f"{prefix}id.npy"), np.load(d / f"{prefix}mu.npy"), np.load(d / f"{prefix}log_scale.npy"),
                   np.load(d / f"{prefix}rotation.npy"), np.load(d / f"{prefix}opacity_logit.npy"),
                   np.load(d / f"{prefix}sh.npy"))

    def copy(self) -> "Splats":
        return Splats(self.id.copy(), self.mu.copy(), self.log_scale.copy(), self.rotation.copy(),
                      self.opacity_logit.copy(), self.sh.copy())

    def take(self, idx) -> "Splats":
        idx = np.asarray(idx)
        return Splats(np.ascontiguousarray(self.id[idx]), np.ascontiguousarray(self.mu[idx]),
                      np.ascontiguousarray(self.log_scale[idx]), np.ascontiguousarray(self.rotation[idx]),
                      np.ascontiguousarray(self.opacity_logit[idx]), np.ascontiguousarray(self.sh[idx]))

    def c(self) -> capi.SplatsC:
        for a in (self.id, self.mu, self.log_scale, self.rotation, self.opacity_logit, self.sh):
            assert a.flags["C_CONTIGUOUS"]
        s = capi.SplatsC()
        s.n = self.n
        s.sh_coeffs = self.sh_coeffs
        s.id = self.id.ctypes.data_as(C.POINTER(C.c_uint64))
        s.mu, s.log_scale, s.rotation = fptr(self.mu), fptr(self.log_scale), fptr(self.rotation)
        s.opacity_logit, s.sh = fptr(self.opacity_logit), fptr(self.sh)
        return s

    def flat(self) -> np.ndarray:
        """All 59 (or 11+3C) parameters per splat, concatenated in GradBuffers order."""
        n = self.n
        return np.concatenate([self.mu, self.log_scale, self.rotation, self.opacity_logit[:, None],
                               self.sh.reshape(n, -1)], axis=1)


def synth_splats(count: int, clustered: bool = False, sh_degree: int = 3, extent: float = 1.0,
                 seed: int = 11) -> Splats:
    """synth_scene's ground-truth splats (io.hpp:491-537), bit-identical streams."""
    s = Splats.empty(count, (sh_degree + 1) ** 2)
    cs = s.c()
    check(lib().dgs_synth_splats(count, int(clustered), sh_degree, extent, seed, C.byref(cs)))
    return s


def ring_camera(width: int, height: int, i: int, n_views: int = 64, fov_deg: float = 60.0,
                ring_radius: float = 3.2, extent: float = 1.0) -> Camera:
    cam = Camera()
    check(lib().dgs_ring_camera(width, height, fov_deg, ring_radius, extent, n_views, i, C.byref(cam)))
    return cam


def save_splats_ply(splats: Splats, path: str, binary: bool = True) -> None:
    """io.hpp:257-297 (3DGS property convention, float32)."""
    sc = splats.c()
    check(lib().dgs_save_splats_ply(C.byref(sc), str(path).encode(), int(binary)))


def load_splats_ply(path: str) -> Splats:
    """load_ply's splat mode (io.hpp:85-255); ids 0..n-1."""
    n, shc = C.c_int64(), C.c_int32()
    check(lib().dgs_load_splats_ply(str(path).encode(), None, C.byref(n), C.byref(shc)))
    out = Splats.empty(int(n.value), int(shc.value))
    oc = out.c()
    check(lib().dgs_load_splats_ply(str(path).encode(), C.byref(oc), None, None))
    return out


def init_from_pointcloud(ctx: "Context", points: np.ndarray, colors: np.ndarray | None, target_count: int,
                         seed: int, sh_degree: int = 3) -> Splats:
    """trainer.hpp:24-91 init_from_pointcloud; the 3-nearest-neighbour term runs
    on ctx's GPU (exact k-NN on a uniform grid instead of O(N^2))."""
    points = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
    cols = None if colors is None else np.ascontiguousarray(colors, np.float32).reshape(-1, 3)
    out = Splats.empty(int(target_count), (sh_degree + 1) ** 2)
    oc = out.c()
    check(lib().dgs_init_from_pointcloud(ctx.handle, ptr(points), points.shape[0], ptr(cols),
                                         0 if cols is None else cols.shape[0], int(target_count), int(seed),
                                         int(sh_degree), C.byref(oc)))
    return out


def perturb(splats: Splats, seed: int) -> Splats:
    s = splats.copy()
    cs = s.c()
    check(lib().dgs_perturb_splats(C.byref(cs), seed))
    return s


# ---------------------------------------------------------------------------
# Partition (partition.hpp)
# ---------------------------------------------------------------------------
@dataclass
class PartitionTable:
    planes: np.ndarray   # structured copy: [K, depth, 5] = (n0, n1, n2, d, closed)
    depth: int

    @property
    def subset_count(self) -> int:
        return int(self.planes.shape[0])

    def c_planes(self):
        K, L = self.planes.shape[0], self.planes.shape[1]
        arr = (Plane * max(K * L, 1))()
        for k in range(K):
            for j in range(L):
                p = arr[k * L + j]
                p.n[0], p.n[1], p.n[2], p.d = (float(x) for x in self.planes[k, j, :4])
                p.closed = int(self.planes[k, j, 4])
        return arr

    def locate(self, x: np.ndarray) -> np.ndarray:
        """partition.hpp:66-71 for a batch of points (float32 semantics)."""
        x = np.asarray(x, np.float32)
        out = np.full(x.shape[0], -1, np.int64)
        for k in range(self.subset_count):
            inside = np.ones(x.shape[0], bool)
            for j in range(self.planes.shape[1]):
                n = self.planes[k, j, :3].astype(np.float32)
                v = (n[0] * x[:, 0] + (n[1] * x[:, 1] + n[2] * x[:, 2])) + np.float32(self.planes[k, j, 3])
                inside &= (v <= 0) if self.planes[k, j, 4] else (v < 0)
            out[(out < 0) & inside] = k
        return out


def slice_plan(height: int, slices: int, s: int) -> tuple[int, int, int, int]:
    """(r0, r1, h0, h1): owned pixel rows and the 10-row SSIM halo of slice s."""
    out = np.zeros(4, np.int32)
    check(lib().dgs_slice_plan(height, slices, s, ptr(out)))
    return tuple(int(x) for x in out)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) through the C-ABI; rank 0 creates it, the
    caller broadcasts it (torch.distributed) before building the Managers."""
    buf = C.create_string_buffer(128)
    check(lib().dgs_nccl_unique_id(buf))
    return buf.raw


def subset_owner(k: int, k_count: int, world: int) -> int:
    return int(lib().dgs_subset_owner(k, k_count, world))


def build_kdtree(centers: np.ndarray, depth: int) -> PartitionTable:
    centers = np.ascontiguousarray(centers, dtype=np.float32)
    K = 1 << depth
    arr = (Plane * max(K * depth, 1))()
    check(lib().dgs_build_kdtree(ptr(centers), centers.shape[0], depth, arr))
    planes = np.zeros((K, depth, 5), np.float32)
    for k in range(K):
        for j in range(depth):
            p = arr[k * depth + j]
            planes[k, j] = (p.n[0], p.n[1], p.n[2], p.d, p.closed)
    return PartitionTable(planes, depth)


def assign_subsets(table: PartitionTable, splats: Splats, d_multiplier: float = 3.0) -> list[np.ndarray]:
    """N_k as indices into `splats`, input order (partition.hpp:234-251)."""
    K, L = table.planes.shape[0], table.planes.shape[1]
    mask = np.zeros((splats.n, K), np.uint8)
    check(lib().dgs_assign_subsets(table.c_planes(), K, L, ptr(splats.mu), ptr(splats.log_scale), splats.n,
                                   d_multiplier, ptr(mask)))
    return [np.nonzero(mask[:, k])[0] for k in range(K)]


# ---------------------------------------------------------------------------
# Device context
# ---------------------------------------------------------------------------
class Context:
    """One dgs_ctx (one GPU / rank).  Owns subset state in HBM."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 transport=None):
        """transport: an object with send/recv/flush/allreduce methods (e.g.
        paper_2406_11836_b200/host_transport.py) replacing NCCL for the multi-rank exchange."""
        self._h = C.c_void_p()
        self._transport = None
        if transport is not None:
            t = capi.HostTransportC()
            t.user = None
            t.send = capi.XFER_SEND(transport.send)
            t.recv = capi.XFER_RECV(transport.recv)
            t.flush = capi.XFER_FLUSH(transport.flush)
            t.allreduce_sum_f64 = capi.XFER_ALLREDUCE(transport.allreduce)
            self._transport = (transport, t)  # keep the callbacks alive
            check(lib().dgs_ctx_create_host_transport(device, rank, world, C.byref(t), C.byref(self._h)))
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            check(lib().dgs_ctx_create(device, rank, world, idbuf, C.byref(self._h)))
        self.table: PartitionTable | None = None

    def close(self):
        if self._h:
            check(lib().dgs_ctx_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        return lib().dgs_stream(self._h) or 0

    def set_graph_mode(self, on: bool):
        """Train steps as CUDA graph replays (dgs_set_graph_mode)."""
        check(lib().dgs_set_graph_mode(self._h, int(on)))

    def save_state(self):
        """Rollback point in HBM for every local subset (dgs_state_save)."""
        check(lib().dgs_state_save(self._h))

    def restore_state(self):
        """Back to the last save_state, in place (dgs_state_restore)."""
        check(lib().dgs_state_restore(self._h))

    def sync(self):
        check(lib().dgs_sync(self._h))

    def set_collect_stats(self, on: bool):
        check(lib().dgs_set_collect_stats(self._h, int(on)))

    def set_backward_records(self, on: bool):
        check(lib().dgs_set_backward_records(self._h, int(on)))

    def set_profiling(self, on: bool):
        check(lib().dgs_set_profiling(self._h, int(on)))

    def stage_times(self) -> dict:
        ms = np.zeros(len(capi.STAGES), np.float64)
        cnt = np.zeros(len(capi.STAGES), np.uint64)
        check(lib().dgs_stage_times(self._h, ptr(ms), ptr(cnt)))
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(capi.STAGES)}

    def set_table(self, table: PartitionTable):
        self.table = table
        check(lib().dgs_set_table(self._h, table.c_planes(), table.subset_count, table.planes.shape[1]))

    def set_epoch(self, epoch: int):
        """The manager's partition epoch: local subsets loaded with another
        epoch are refused with "partition epoch mismatch" (worker.hpp:63)."""
        check(lib().dgs_set_epoch(self._h, int(epoch)))

    def set_options(self, ro: capi.RenderOptionsC | None = None, cfg: capi.TrainConfigC | None = None):
        check(lib().dgs_set_options(self._h, C.byref(ro) if ro is not None else None,
                                    C.byref(cfg) if cfg is not None else None))

    def load_subset(self, k: int, params: Splats, m: Splats | None = None, v: Splats | None = None,
                    adam_step: int = 0, epoch: int = 0):
        pc = params.c()
        mc = m.c() if m is not None else None
        vc = v.c() if v is not None else None
        check(lib().dgs_subset_load(self._h, k, C.byref(pc), C.byref(mc) if mc else None,
                                    C.byref(vc) if vc else None, adam_step, epoch))

    def store_subset(self, k: int, sh_coeffs: int) -> tuple[Splats, Splats, Splats, int]:
        n = lib().dgs_subset_size(self._h, k)
        if n < 0:
            raise ValueError(f"subset {k} is not loaded on this rank")
        p, m, v = Splats.empty(n, sh_coeffs), Splats.empty(n, sh_coeffs), Splats.empty(n, sh_coeffs)
        pc, mc, vc = p.c(), m.c(), v.c()
        step = C.c_uint64()
        check(lib().dgs_subset_store(self._h, k, C.byref(pc), C.byref(mc), C.byref(vc), C.byref(step)))
        m.id[:] = p.id
        v.id[:] = p.id
        return p, m, v, int(step.value)

    # -- per-subset forward / backward --------------------------------------
    def render_partial(self, k: int, cam: Camera, dbg_cap: int = 0):
        px = cam.width * cam.height
        ct = np.zeros((cam.height, cam.width, 4), np.float32)
        ids = np.zeros(px * dbg_cap, np.uint32) if dbg_cap else None
        cnt = np.zeros(px, np.uint32) if dbg_cap else None
        check(lib().dgs_render_partial(self._h, k, C.byref(cam), ptr(ct), dbg_cap, ptr(ids), ptr(cnt)))
        if dbg_cap:
            return ct, ids.reshape(px, dbg_cap), cnt
        return ct

    def dump_bins(self, k: int, cam: Camera, cap: int | None = None):
        tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        n_pairs = C.c_int64()
        off = np.zeros(tiles + 1, np.int64)
        cap = cap or 1
        ent = np.zeros(cap, np.int32)
        rc = lib().dgs_dump_bins(self._h, k, ptr(off), ptr(ent), cap, C.byref(n_pairs))
        if rc != 0 and n_pairs.value > cap:
            ent = np.zeros(n_pairs.value, np.int32)
            rc = lib().dgs_dump_bins(self._h, k, ptr(off), ptr(ent), n_pairs.value, C.byref(n_pairs))
        check(rc)
        return off, ent[: n_pairs.value]

    def dump_records(self, k: int):
        n = lib().dgs_subset_size(self._h, k)
        recs = np.zeros((n, 16), np.float32)
        counts = np.zeros(n, np.uint32)
        check(lib().dgs_dump_records(self._h, k, ptr(recs), ptr(counts)))
        return recs, counts

    def render_partial_backward(self, k: int, cam: Camera, grad_ct: np.ndarray, sh_coeffs: int) -> Splats:
        n = lib().dgs_subset_size(self._h, k)
        g = Splats.empty(n, sh_coeffs)
        gc = g.c()
        grad_ct = np.ascontiguousarray(grad_ct, np.float32)
        check(lib().dgs_render_partial_backward(self._h, k, C.byref(cam), ptr(grad_ct), C.byref(gc)))
        return g

    def dump_pixel_grads(self, k: int) -> np.ndarray:
        n = lib().dgs_subset_size(self._h, k)
        out = np.zeros((n, 9), np.float32)
        check(lib().dgs_dump_pixel_grads(self._h, k, ptr(out)))
        return out

    def adam_apply(self, k: int, grads: Splats):
        gc = grads.c()
        check(lib().dgs_adam_apply(self._h, k, C.byref(gc)))

    # -- manager side ----------------------------------------------------------
    def pixel_orders(self, cam: Camera):
        K = self.table.subset_count
        order = np.zeros((cam.height, cam.width, K), np.uint16)
        count = np.zeros((cam.height, cam.width), np.uint16)
        check(lib().dgs_pixel_orders(self._h, C.byref(cam), ptr(order), ptr(count)))
        return order, count

    def merge(self, cam: Camera, partials: np.ndarray, bg=(0.0, 0.0, 0.0)):
        partials = np.ascontiguousarray(partials, np.float32)
        bga = np.asarray(bg, np.float32)
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        t = np.zeros((cam.height, cam.width), np.float32)
        check(lib().dgs_merge(self._h, C.byref(cam), ptr(partials), ptr(bga), ptr(rgb), ptr(t)))
        return rgb, t

    def loss(self, render: np.ndarray, target: np.ndarray, lam: float = 0.2, inv_batch: float = 1.0):
        render = np.ascontiguousarray(render, np.float32)
        target = np.ascontiguousarray(target, np.float32)
        if render.shape != target.shape:
            raise ValueError("loss: resolution mismatch")
        H, W = render.shape[:2]
        grad = np.zeros_like(render)
        val = C.c_double()
        sums = np.zeros(3, np.float64)
        check(lib().dgs_loss(self._h, W, H, ptr(render), ptr(target), lam, inv_batch, ptr(grad), C.byref(val),
                             ptr(sums)))
        return float(val.value), grad, sums

    def merge_backward(self, cam: Camera, partials: np.ndarray, grad_color: np.ndarray, bg=(0.0, 0.0, 0.0)):
        partials = np.ascontiguousarray(partials, np.float32)
        grad_color = np.ascontiguousarray(grad_color, np.float32)
        bga = np.asarray(bg, np.float32)
        out = np.zeros_like(partials)
        check(lib().dgs_merge_backward(self._h, C.byref(cam), ptr(partials), ptr(grad_color), ptr(bga), ptr(out)))
        return out

    def render(self, cam: Camera, bg=(0.0, 0.0, 0.0)):
        bga = np.asarray(bg, np.float32)
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        t = np.zeros((cam.height, cam.width), np.float32)
        check(lib().dgs_render(self._h, C.byref(cam), ptr(bga), ptr(rgb), ptr(t)))
        return rgb, t

    def set_virtual_slices(self, slices: int):
        check(lib().dgs_set_virtual_slices(self._h, slices))

    def dump_grad_maps(self, k: int, view: int, cam: Camera):
        ct = np.zeros((cam.height, cam.width, 4), np.float32)
        g = np.zeros((cam.height, cam.width, 4), np.float32)
        check(lib().dgs_dump_grad_maps(self._h, k, view, ptr(ct), ptr(g)))
        return ct, g

    def upload_targets(self, targets: np.ndarray) -> int:
        targets = np.ascontiguousarray(targets, np.float32)
        B, H, W, _ = targets.shape
        dp = C.c_void_p()
        check(lib().dgs_upload_targets(self._h, B, W, H, ptr(targets), C.byref(dp)))
        return dp.value

    def train_step(self, cams, targets, bg=(0.0, 0.0, 0.0), targets_device_ptr: int | None = None) -> dict:
        cams = list(cams)
        arr = (Camera * len(cams))(*cams)
        bga = np.asarray(bg, np.float32)
        res = StepResult()
        if targets_device_ptr is not None:
            check(lib().dgs_train_step(self._h, len(cams), arr, C.c_void_p(targets_device_ptr), 1, ptr(bga),
                                       C.byref(res)))
        else:
            t = np.ascontiguousarray(targets, np.float32)
            check(lib().dgs_train_step(self._h, len(cams), arr, ptr(t), 0, ptr(bga), C.byref(res)))
        return res.as_dict()


class Manager:
    """Manager<float> (manager.hpp:212-516) on one process: KD partition on the
    host (bit-exact), every subset resident on this rank's GPU."""

    def __init__(self, splats: Splats, config: capi.TrainConfigC | None = None,
                 options: capi.RenderOptionsC | None = None, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, transport=None):
        """world > 1: one Manager per rank (one process per GPU).  Every rank
        builds the same KD table on the host (bit-exact, deterministic) and
        loads only the subsets it owns (`subset_owner`, contiguous blocks);
        `train_step` then exchanges partial rows and their gradients over the
        context's NCCL communicator (`nccl_id` from `nccl_unique_id()` on rank
        0, broadcast by the caller)."""
        self.config = config if config is not None else train_config()
        self.options = options if options is not None else render_options()
        if world > 1 and nccl_id is None and transport is None:
            raise ValueError("Manager: world > 1 needs the NCCL unique id of rank 0")
        self.rank, self.world = rank, world
        self.ctx = Context(device, rank, world, nccl_id, transport)
        self.sh_coeffs = splats.sh_coeffs
        self.ids = np.sort(splats.id.copy())
        self._distribute(splats, epoch=0)

    def _distribute(self, splats: Splats, epoch: int, m: Splats | None = None, v: Splats | None = None,
                    adam_step: int = 0):
        self.table = build_kdtree(splats.mu, int(self.config.kd_depth))
        self.members = assign_subsets(self.table, splats, float(self.options.truncation_radius))
        self.ctx.set_table(self.table)
        self.ctx.set_options(self.options, self.config)
        K = self.table.subset_count
        if K < self.world:
            raise ValueError(f"Manager: {K} KD subsets cannot cover {self.world} ranks (kd_depth too small)")
        for k, idx in enumerate(self.members):
            if subset_owner(k, K, self.world) != self.rank:
                continue
            self.ctx.load_subset(k, splats.take(idx), m.take(idx) if m is not None else None,
                                 v.take(idx) if v is not None else None, adam_step=adam_step, epoch=epoch)
        self.ctx.set_epoch(epoch)
        self.epoch = epoch

    def train_step(self, cams, targets, bg=(0.0, 0.0, 0.0), targets_device_ptr=None) -> dict:
        return self.ctx.train_step(cams, targets, bg, targets_device_ptr)

    def render(self, cam: Camera, bg=(0.0, 0.0, 0.0)):
        return self.ctx.render(cam, bg)

    def snapshot(self):
        """manager.hpp:390-418: gather every subset's (p, m, v); a shared splat
        resolves to the replica held by the subspace containing its centre, else
        to the lowest subset index.  Returned in id order (the reference returns
        owner-resolved packs first, then the rest).  world > 1: every rank sends
        its owned subsets to rank 0 over torch.distributed (the process group
        the caller initialised, NCCL or gloo); rank 0 returns the snapshot and
        the other ranks None (the reference's snapshot lives on the manager)."""
        parts = {k: self.ctx.store_subset(k, self.sh_coeffs) for k in range(self.table.subset_count)
                 if subset_owner(k, self.table.subset_count, self.world) == self.rank}
        if self.world > 1:
            import torch.distributed as dist
            if not dist.is_initialized():
                raise RuntimeError("snapshot: world > 1 needs the torch.distributed process group of the ranks")
            got = [None] * self.world if self.rank == 0 else None
            dist.gather_object(parts, got, dst=0)
            if self.rank != 0:
                return None
            parts = {k: v for d in got for k, v in d.items()}
        K = self.table.subset_count
        if sorted(parts) != list(range(K)):
            raise RuntimeError("snapshot: missing subsets " + str(sorted(set(range(K)) - set(parts))))
        ids = np.concatenate([parts[k][0].id for k in range(K)])
        kk = np.concatenate([np.full(parts[k][0].n, k, np.int64) for k in range(K)])
        owner = np.concatenate([self.table.locate(parts[k][0].mu) == k for k in range(K)])
        pri = np.where(owner, kk, K + kk)  # owner-held replica first, then the lowest k
        order = np.lexsort((pri, ids))
        first = np.ones(len(order), bool)
        first[1:] = ids[order][1:] != ids[order][:-1]
        chosen = order[first]
        if len(chosen) != len(self.ids) or not np.array_equal(ids[chosen], self.ids):
            raise RuntimeError("snapshot lost splats")

        def gather(which):
            out = Splats.empty(len(chosen), self.sh_coeffs)
            for f in ("id", "mu", "log_scale", "rotation", "opacity_logit", "sh"):
                getattr(out, f)[...] = np.concatenate([getattr(parts[k][which], f) for k in range(K)])[chosen]
            return out
        return gather(0), gather(1), gather(2), parts[0][3]

    def checkpoint(self, path: str) -> None:
        """snapshot(checkpoint_path) (manager.hpp:390-396): the merged splats as a
        3DGS PLY (Adam moments are not part of the file format); written by rank 0."""
        snap = self.snapshot()
        if snap is not None:
            save_splats_ply(snap[0], path)

    def repartition(self, device: bool = True):
        """Manager::repartition (manager.hpp:421-430).  device=True (default):
        snapshot, KD build, assignment and migration on the GPU
        (dgs_repartition; across ranks the replica keys and centres are
        all-gathered and the migrating state moves all-to-all); device=False:
        the host path through snapshot() and a reload (single rank)."""
        if not device:
            return self.repartition_host()
        depth = int(self.config.kd_depth)
        K = 1 << depth
        arr = (Plane * max(K * depth, 1))()
        check(lib().dgs_repartition(self.ctx.handle, depth, float(self.options.truncation_radius), len(self.ids),
                                    self.epoch + 1, arr))
        planes = np.zeros((K, depth, 5), np.float32)
        for k in range(K):
            for j in range(depth):
                q = arr[k * depth + j]
                planes[k, j] = (q.n[0], q.n[1], q.n[2], q.d, q.closed)
        self.table = PartitionTable(planes, depth)
        self.ctx.table = self.table
        self.members = None  # membership lives on the device
        self.epoch += 1

    def repartition_host(self):
        p, m, v, step = self.snapshot()
        if not np.array_equal(np.sort(p.id), self.ids):
            raise RuntimeError("repartition checksum mismatch")
        self._distribute(p, self.epoch + 1, m, v, step)

    def close(self):
        self.ctx.close()
