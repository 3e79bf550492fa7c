"""Multi-process (gloo, world_size 2, CPU) checks of the time-slab decomposition's
host logic: slab partition, per-rank frame-addressable input
generation, unique-id broadcast transport, and the decomposition itself --
per-rank halo exchange of r_t frames of p = F*x plus an allreduce of the norm
partials reproduces the single-process oracle (the same phase structure the
C library runs with NCCL)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as WL
from paper_2212_08058_b200.dist import slab_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    errs = [r for r in res if isinstance(r, str)]
    assert not errs, errs
    return sorted(res, key=lambda t: t[0])


def _worker(fn, rank, world, port, q, args):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = fn(rank, world, *args)
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


def test_slab_range_partitions():
    for T in (1, 5, 64, 70, 512):
        for n in (1, 2, 3, 4, 8):
            if n > T:
                continue
            rs = [slab_range(T, n, r) for r in range(n)]
            assert rs[0][0] == 0 and rs[-1][1] == T
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


# ------------------------------------------------------------------ per-rank generation
def _gen(rank, world, name, shape):
    cfg = WL.get_config(name, **shape)
    t0, t1 = slab_range(cfg.T, world, rank)
    wl = WL.generate(name, cfg=cfg, t_range=(t0, t1))
    t = torch.from_numpy(np.ascontiguousarray(wl.ch))
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.shape[2]]))
    mx = max(int(s) for s in sizes)
    pad = torch.zeros(t.shape[:2] + (mx,) + t.shape[3:])
    pad[:, :, : t.shape[2]] = t
    gath = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(gath, pad)
    full = torch.cat([g[:, :, : int(s)] for g, s in zip(gath, sizes)], dim=2)
    return full.numpy()


def test_slab_generation_matches_full():
    shape = dict(T=9, H=40, W=60)
    res = _run(_gen, 2, "c5", shape)
    full = WL.generate("c5", cfg=WL.get_config("c5", **shape)).ch
    for _, got in res:
        np.testing.assert_array_equal(got, full)


# ------------------------------------------------------------------ unique-id transport
def _bcast(rank, world):
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = torch.arange(128, dtype=torch.uint8)
    dist.broadcast(buf, src=0)
    return bytes(buf.tolist())


def test_unique_id_broadcast_transport():
    res = _run(_bcast, 2)
    assert all(r[1] == bytes(range(128)) for r in res)


# ------------------------------------------------------------------ the decomposition
def _slab_solve(rank, world, F_full, rt, rs, sig_t, sig_s, K):
    """Per-rank phases: p = F*x -> halo exchange of rt frames -> temporal pass over
    [halo_lo, local, halo_hi] -> spatial passes -> y = F*u -> allreduce sum(y^2) -> x = y/nu."""
    T = F_full.shape[1]
    t0, t1 = slab_range(T, world, rank)
    F = F_full[:, t0:t1]
    gt, gs = O.gaussian_taps(sig_t, rt), O.gaussian_taps(sig_s, rs)
    x = F.copy()
    nus = []
    for _ in range(K):
        p = F * x
        lo = np.zeros_like(p[:, :rt])
        hi = np.zeros_like(p[:, :rt])
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(p[:, :rt])), rank - 1))
            buf_lo = torch.zeros(p[:, :rt].shape, dtype=torch.float64)
            reqs.append(dist.irecv(buf_lo, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(p[:, -rt:])), rank + 1))
            buf_hi = torch.zeros(p[:, -rt:].shape, dtype=torch.float64)
            reqs.append(dist.irecv(buf_hi, rank + 1))
        for r in reqs:
            r.wait()
        if rank > 0:
            lo = buf_lo.numpy()
        if rank < world - 1:
            hi = buf_hi.numpy()
        ext = np.concatenate([lo, p, hi], axis=1)          # frames t0-rt .. t1+rt
        u = np.empty_like(p)
        for b in range(p.shape[0]):
            v = O.correlate_axis(ext[b], gt, 0)[rt:rt + p.shape[1]]
            u[b] = O.correlate_axis(O.correlate_axis(v, gs, 1), gs, 2)
        y = F * u
        ss = torch.tensor([float(np.sum(y[b] ** 2)) for b in range(y.shape[0])], dtype=torch.float64)
        dist.all_reduce(ss)
        nu = np.sqrt(ss.numpy())
        nus.append(nu)
        x = y / nu[:, None, None, None]
    return t0, x, np.array(nus).T


@pytest.mark.parametrize("world,T", [(2, 11)])
def test_slab_decomposition_equals_oracle(world, T):
    rng = np.random.default_rng(3)
    F = rng.random((2, T, 12, 14)) * 0.8 + 0.1
    rt, rs, K = 2, 3, 4
    res = _run(_slab_solve, world, F, rt, rs, 1.0, 1.2, K)
    xo, st = O.power_iterate(F, O.gaussian_taps(1.0, rt), O.gaussian_taps(1.2, rs), K)
    x = np.concatenate([r[1][1] for r in res], axis=1)
    np.testing.assert_allclose(x, xo, rtol=0, atol=1e-13)
    for r in res:
        np.testing.assert_allclose(r[1][2], st["nu"], rtol=1e-13)


def _frames(ranges):
    out = []
    for t0, n in ranges:
        out.extend(range(t0, t0 + n))
    return out


def test_overlapped_schedule_launch_ranges():
    """The overlapped schedule's spatial-pass launches (the library's own host logic,
    sfseg_slab_launch_ranges) tile the slab exactly once, and every frame a neighbour needs
    as halo is computed before the exchange; thin slabs collapse to one launch."""
    from paper_2212_08058_b200.dist import slab_launch_ranges
    for T in (1, 5, 6, 7, 12, 13, 19, 64, 70):
        for RT in (0, 1, 3, 6, 9):
            for lo in (False, True):
                for hi in (False, True):
                    rg, nb = slab_launch_ranges(T, RT, lo, hi)
                    fr = _frames(rg)
                    assert sorted(fr) == list(range(T)) and len(fr) == T, (T, RT, lo, hi, rg)
                    assert 1 <= nb <= len(rg) and all(n > 0 for _, n in rg)
                    before = set(_frames(rg[:nb]))
                    need = set()
                    if lo:
                        need |= set(range(min(RT, T)))
                    if hi:
                        need |= set(range(max(0, T - RT), T))
                    assert need <= before, (T, RT, lo, hi, rg, nb)
                    if 0 < (RT if lo else 0) + (RT if hi else 0) < T:
                        assert len(rg) == nb + 1     # an interior launch overlaps the exchange
                    else:
                        assert rg == [(0, T)] and nb == 1


def _ranges_rank(rank, world, T_global, RT):
    from paper_2212_08058_b200.dist import slab_launch_ranges
    t0, t1 = slab_range(T_global, world, rank)
    rg, nb = slab_launch_ranges(t1 - t0, RT, rank > 0, rank < world - 1)
    # global frames this rank computes before its exchange, and the halo frames it receives
    sent = sorted(t0 + f for f in _frames(rg[:nb]))
    recv = []
    if rank > 0:
        recv += list(range(t0 - RT, t0))
    if rank < world - 1:
        recv += list(range(t1, t1 + RT))
    g = [None] * world
    dist.all_gather_object(g, (sent, recv))
    # every halo frame a rank receives was computed by its owner before the owner's exchange
    for r in range(world):
        owner_sent = set().union(*[set(g[o][0]) for o in range(world) if o != r])
        assert set(g[r][1]) <= owner_sent, (r, g)
    return True


@pytest.mark.parametrize("world,T,RT", [(2, 70, 6), (3, 64, 9), (4, 40, 6)])
def test_overlapped_schedule_halo_frames_ready_before_exchange(world, T, RT):
    assert all(r[1] for r in _run(_ranges_rank, world, T, RT))
