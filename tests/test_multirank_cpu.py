"""CPU, world_size 2 (gloo): the multi-rank step's host logic — KD subset
ownership, pixel-row slices with the 10-row SSIM halo, the forward all-to-all
of partial rows and the backward return of (dL/dC_k, dL/dT_k) — executed by
two real processes.  Per-rank compute uses the C restatement of the
reference (oracle/dgs_oracle.c, the checker); the plan comes from the
product's C-ABI (dgs_slice_plan, dgs_subset_owner).  The distributed result
must equal the single-process merge/loss/adjoint bit for bit."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_binding as ob
from conftest import Golden

NAME = "g4_synth_kd3_bg"  # 8 subsets, non-zero background


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_inputs():
    g = Golden(NAME)
    s = g.splats()
    planes = g["kd_planes"].reshape(-1, 5)
    depth = g.args["kd"]
    K = 1 << depth
    subs = [ob.subspace(planes[k * depth:(k + 1) * depth]) for k in range(K)]
    off, ids = g["kd_member_off"], g["kd_member_ids"]
    members = [s.take(ids[off[k]:off[k + 1]].astype(np.int64)) for k in range(K)]
    cam = ob.cam_of(g["scene_cameras"][g.args["view"]])
    return g, subs, members, cam, ob.opts(g.oracle_mode)


def _partial(members, subs, cam, o, k):
    sc = ob.Scene(members[k])
    ct = np.zeros((cam.height, cam.width, 4), np.float32)
    ob.lib().orc_partial_render(C.byref(sc.c), C.byref(subs[k]), C.byref(cam), C.byref(o), ob.p(ct), 0, None, None)
    return ct


def _manager_rows(g, subs, cam, partials_win, h0, h1, r0, r1):
    """merge + loss + merge_backward for rows [r0, r1) given partial rows [h0, h1)."""
    K = len(subs)
    H, W = cam.height, cam.width
    order = np.zeros((H, W, K), np.uint16)
    count = np.zeros((H, W), np.uint16)
    arr = (ob.Sub * K)(*subs)
    ob.lib().orc_pixel_orders(arr, K, C.byref(cam), ob.p(order), ob.p(count))
    hr = h1 - h0
    o_w = np.ascontiguousarray(order[h0:h1])
    c_w = np.ascontiguousarray(count[h0:h1])
    bg = np.asarray(g.bg, np.float32)
    rgb = np.zeros((hr, W, 3), np.float32)
    ob.lib().orc_merge(ob.p(partials_win), ob.p(o_w), ob.p(c_w), K, W, hr, ob.p(bg), ob.p(rgb), None)
    return rgb, o_w, c_w, bg


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_11836_b200 import engine
        g, subs, members, cam, o = _oracle_inputs()
        K, H, W = len(subs), cam.height, cam.width
        local = [k for k in range(K) if engine.subset_owner(k, K, world) == rank]
        parts = {k: _partial(members, subs, cam, o, k) for k in local}
        plans = [engine.slice_plan(H, world, j) for j in range(world)]
        r0, r1, h0, h1 = plans[rank]
        # forward all-to-all: rows [h0_j, h1_j) of my subsets to rank j
        win = np.zeros((K, h1 - h0, W, 4), np.float32)
        for k in range(K):
            src = engine.subset_owner(k, K, world)
            for j in range(world):
                jr0, jr1, jh0, jh1 = plans[j]
                if src == rank and j == rank:
                    win[k] = parts[k][jh0:jh1]
                elif src == rank:
                    dist.send(torch.from_numpy(np.ascontiguousarray(parts[k][jh0:jh1])), dst=j)
                elif j == rank:
                    buf = torch.empty((h1 - h0, W, 4), dtype=torch.float32)
                    dist.recv(buf, src=src)
                    win[k] = buf.numpy()
        rgb, o_w, c_w, bg = _manager_rows(g, subs, cam, np.ascontiguousarray(win), h0, h1, r0, r1)
        # merged rows of my slice equal the reference's merged image
        ok_merge = np.array_equal(rgb[r0 - h0:r1 - h0], g["step_render"][r0:r1])
        # merge adjoint for my owned rows (the reference's loss gradient as input)
        gc = np.ascontiguousarray(g["step_grad_color"][h0:h1])
        out = np.zeros_like(win)
        ob.lib().orc_merge_backward(ob.p(np.ascontiguousarray(win)), ob.p(o_w), ob.p(c_w), K, W, h1 - h0, ob.p(gc),
                                    ob.p(bg), ob.p(out))
        # backward: rows [r0_j, r1_j) of every subset back to its owner
        grads = {k: np.zeros((H, W, 4), np.float32) for k in local}
        for k in range(K):
            dst = engine.subset_owner(k, K, world)
            for j in range(world):
                jr0, jr1, jh0, jh1 = plans[j]
                if j == rank and dst == rank:
                    grads[k][r0:r1] = out[k][r0 - h0:r1 - h0]
                elif j == rank:
                    dist.send(torch.from_numpy(np.ascontiguousarray(out[k][r0 - h0:r1 - h0])), dst=dst)
                elif dst == rank:
                    buf = torch.empty((jr1 - jr0, W, 4), dtype=torch.float32)
                    dist.recv(buf, src=j)
                    grads[k][jr0:jr1] = buf.numpy()
        ok_grad = all(np.array_equal(grads[k][..., :3], g[f"k{k}_dC"]) and
                      np.array_equal(grads[k][..., 3], g[f"k{k}_dT"]) for k in local)
        q.put((rank, bool(ok_merge), bool(ok_grad), local))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_plan_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    owned = sorted(k for r in res for k in r[3])
    assert owned == list(range(8))
    for rank, ok_merge, ok_grad, _ in res:
        assert ok_merge, f"rank {rank}: merged slice differs from the reference"
        assert ok_grad, f"rank {rank}: returned partial-map gradients differ from the reference"


def test_slice_plan_covers_image_with_halo():
    from paper_2406_11836_b200 import engine
    for H in (1, 7, 48, 1080, 2160):
        for S in (1, 2, 3, 4, 8):
            if S > H:
                continue
            rows = [engine.slice_plan(H, S, s) for s in range(S)]
            assert rows[0][0] == 0 and rows[-1][1] == H
            for a, b in zip(rows, rows[1:]):
                assert a[1] == b[0]
            for r0, r1, h0, h1 in rows:
                assert h0 == max(0, r0 - 10) and h1 == min(H, r1 + 10)
    assert [engine.subset_owner(k, 8, 2) for k in range(8)] == [0, 0, 0, 0, 1, 1, 1, 1]
    assert [engine.subset_owner(k, 8, 8) for k in range(8)] == list(range(8))
