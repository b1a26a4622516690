"""Slab decomposition host logic: world size 2 over gloo on CPU.

The distributed algorithm of paper_2311_13049_b200/slab.py runs with numpy
stand-ins for the three device stages; it must reproduce the single-process
(P = 1) result bit for bit -- every line transform is the same -- and agree with
the C oracle at the fp64 floor.  The device stages themselves are checked against
the single-GPU apply in tests/test_gpu_parity.py (P = 1 on one B200; this run
has one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_2311_13049_b200 import configs as cfgs
from paper_2311_13049_b200.slab import SlabApply, SlabGeometry


class NumpyStages:
    """numpy restatement of fw_stage_r2c / fw_stage_c2c / fw_stage_c2r_accum semantics."""

    contig = staticmethod(np.ascontiguousarray)

    @staticmethod
    def concat(xs, axis):
        return np.concatenate(xs, axis=axis)

    @staticmethod
    def r2c(x, shape):
        return np.fft.rfft(np.asarray(x).reshape(shape), axis=2)

    @staticmethod
    def c2c(src, shape, axis, dir, w=None, nterms=1, src_ts=0, w_ts=0, scale=1.0):
        outs = []
        for t in range(nterms):
            s = src[t] if (src_ts and src.ndim == 4) else src
            if w is not None:
                s = s * (w[t] if w_ts else w[0])
            n = s.shape[axis]
            o = np.fft.fft(s, axis=axis) if dir < 0 else np.fft.ifft(s, axis=axis) * n
            if scale != 1.0:
                o = o * scale
            outs.append(o)
        return np.stack(outs) if nterms > 1 else outs[0]

    @staticmethod
    def c2r(src, shape, m_first, m_last, dev1):
        out = np.zeros(shape)
        dm = None
        for m in range(m_first, m_last + 1):
            s = src[m - m_first] if src.ndim == 4 else src
            x = np.fft.irfft(s, n=shape[2], axis=2) * shape[2]
            if m >= 1:
                dm = dev1 if m == 1 else dm * dev1
                x = dm * x
            out = out + x
        return out


def tables(J, lo, hi, s, M):
    mu2 = O.port_mu2(J, lo, hi)
    s0 = O.port_order_stats(s)[0]
    H = J[2] // 2 + 1
    m2 = mu2[:, :, :H]
    pos = m2 > 0
    base = np.where(pos, np.power(np.where(pos, m2, 1.0), s0), 0.0)
    L = np.where(pos, np.log(np.where(pos, m2, 1.0)), 0.0)
    w = np.empty((M + 1,) + m2.shape)
    lw = np.zeros_like(m2)
    w[0] = base
    for m in range(1, M + 1):
        lw = np.where(pos, L if m == 1 else lw * L / m, 0.0)
        w[m] = base * lw
    return w, s - s0


class GlooComm:
    def all_to_all(self, blocks):
        send = [torch.from_numpy(np.ascontiguousarray(b)).contiguous() for b in blocks]
        shape = send[0].shape
        flat = torch.stack([torch.view_as_real(b).reshape(-1) if b.is_complex() else b.reshape(-1) for b in send])
        recv = torch.empty_like(flat)
        dist.all_to_all_single(recv, flat)
        out = []
        for p in range(len(blocks)):
            r = recv[p]
            if send[0].is_complex():
                r = torch.view_as_complex(r.reshape(shape + (2,)))
            out.append(r.reshape(shape).numpy())
        return out


def _worker(rank, world, port, J, lo, hi, M, m_first, result_q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    s = 1.0 + 0.3 * np.sin(np.pi * cfgs._mesh(lo, hi, J)[0] / 2.0)
    u = rng.standard_normal(J)
    w, dev1 = tables(J, lo, hi, s, M)
    geo = SlabGeometry(J, world, rank)
    sa = SlabApply(geo, NumpyStages(), GlooComm(), np.ascontiguousarray(w[:, :, geo.cols, :]), dev1[geo.rows], M)
    part = sa.apply(u[geo.rows], m_first)
    parts = [torch.zeros((J[0] // world,) + J[1:], dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(part)))
    if rank == 0:
        result_q.put(np.concatenate([p.numpy() for p in parts]))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def run_distributed(world, J, lo, hi, M, m_first=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, J, lo, hi, M, m_first, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("m_first", [0, 1])
def test_slab_world2_bitwise_equals_single_and_matches_oracle(m_first):
    J, lo, hi, M = (8, 16, 16), (-2.0, -2.0, -2.0), (2.0, 2.0, 2.0), 6
    one = run_distributed(1, J, lo, hi, M, m_first)
    two = run_distributed(2, J, lo, hi, M, m_first)
    assert np.array_equal(one, two)
    rng = np.random.default_rng(5)
    s = 1.0 + 0.3 * np.sin(np.pi * cfgs._mesh(lo, hi, J)[0] / 2.0)
    u = rng.standard_normal(J)
    ref, _ = O.port_apply(J, lo, hi, s, u, M, m_first=m_first)
    assert np.linalg.norm(two - ref) / np.linalg.norm(ref) < 1e-13


def test_slab_geometry_validation():
    with pytest.raises(ValueError):
        SlabGeometry((12, 16, 16), 8, 0)
    g = SlabGeometry((256, 256, 256), 8, 3)
    assert (g.J0l, g.J1l, g.H) == (32, 32, 129)
    assert g.rows == slice(96, 128) and g.cols == slice(96, 128)


def test_slab_world2_single_term():
    """One term in the inverse (M = 1, m_first = 1): the batched transpose keeps its term axis."""
    J, lo, hi, M = (8, 16, 16), (-2.0, -2.0, -2.0), (2.0, 2.0, 2.0), 1
    two = run_distributed(2, J, lo, hi, M, 1)
    rng = np.random.default_rng(5)
    s = 1.0 + 0.3 * np.sin(np.pi * cfgs._mesh(lo, hi, J)[0] / 2.0)
    u = rng.standard_normal(J)
    ref, _ = O.port_apply(J, lo, hi, s, u, M, m_first=1)
    assert np.linalg.norm(two - ref) / np.linalg.norm(ref) < 1e-13
