"""Slab-decomposed apply of the M-term operator over P ranks (one GPU per rank).

SURVEY.md §8(e): axis 0 of a 3D grid J0 x J1 x J2 is split over P ranks.
Rank r owns physical planes [r J0/P, (r+1) J0/P) and, in the transposed spectral
layout, axis-1 lines [r J1/P, (r+1) J1/P):

  forward   R2C along axis 2 and C2C along axis 1 on the local slab
            -> all-to-all transpose -> C2C along axis 0 (x 1/N)      [J0][J1/P][J2/2+1]
  inverse   for all terms at once: (w_m .* uhat) -> C2C along axis 0
            -> all-to-all transpose back -> C2C along axis 1
            -> per-row C2R with the ascending-m (s-s0)^m recombination  [J0/P][J1][J2]

i.e. (M+2)-term's worth of all-to-alls per apply (one forward, one batched
backward carrying every term), with NO collective anywhere else.  Every 1D line
transform is the one the single-device path performs, so the result is
bit-identical to P = 1 (tests/test_slab.py checks this with world size 2 on CPU,
tests/test_gpu_parity.py checks the device stages against the single-GPU apply).

The local stages are pluggable:
  * ``DeviceStages`` -- the sm_100a kernels through the C-ABI stage entry points
    (fw_stage_r2c / fw_stage_c2c / fw_stage_c2r_accum); buffers are torch CUDA
    tensors on the context's stream; the transpose is torch.distributed
    all_to_all_single (NCCL over NVLink when launched under torchrun on one node).
  * tests supply a numpy implementation of the same three stages to exercise the
    decomposition logic with the gloo backend on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass
class SlabGeometry:
    J: tuple          # global (J0, J1, J2)
    P: int
    rank: int

    def __post_init__(self):
        J0, J1, J2 = self.J
        if J0 % self.P or J1 % self.P:
            raise ValueError(f"axes 0 and 1 ({J0}, {J1}) must be divisible by P = {self.P}")

    @property
    def H(self):
        return self.J[2] // 2 + 1

    @property
    def J0l(self):
        return self.J[0] // self.P

    @property
    def J1l(self):
        return self.J[1] // self.P

    @property
    def N(self):
        return self.J[0] * self.J[1] * self.J[2]

    @property
    def rows(self):  # physical planes owned by this rank
        return slice(self.rank * self.J0l, (self.rank + 1) * self.J0l)

    @property
    def cols(self):  # axis-1 lines owned in the transposed spectral layout
        return slice(self.rank * self.J1l, (self.rank + 1) * self.J1l)


class SlabApply:
    """Distributed M-term apply for one operator.

    stages: object with r2c(x, shape) -> H, c2c(src, shape, axis, dir, w=None, nterms=1,
            src_ts=0, w_ts=0, scale=1.0) -> dst, c2r(src, shape, m_first, m_last, dev1) -> out,
            and array helpers empty/concat/stack (numpy-like semantics on its array type).
    comm:   object with all_to_all(list_of_P_arrays) -> list_of_P_arrays.
    w_local: (M+1, J0, J1/P, H) complex-half weights of this rank's spectral columns.
    dev1_local: (J0/P, J1, J2) values of s - s0 on this rank's planes.
    """

    def __init__(self, geo: SlabGeometry, stages, comm, w_local, dev1_local, m_last: int):
        self.g, self.st, self.comm = geo, stages, comm
        self.w, self.dev1, self.m_last = w_local, dev1_local, m_last

    def forward(self, u_slab):
        g, st = self.g, self.st
        loc = (g.J0l, g.J[1], g.J[2])
        Y = st.r2c(u_slab, loc)                                   # [J0l][J1][H]
        Y = st.c2c(Y, loc, axis=1, dir=-1)
        if g.P == 1:  # no transpose: the local array is the whole spectrum
            T = Y
        else:
            send = [st.contig(Y[:, q * g.J1l:(q + 1) * g.J1l, :]) for q in range(g.P)]
            recv = self.comm.all_to_all(send)                     # from p: [J0l][J1l][H]
            T = st.concat(recv, axis=0)                           # [J0][J1l][H]
        return st.c2c(T, (g.J[0], g.J1l, g.J[2]), axis=0, dir=-1, scale=1.0 / g.N)

    def inverse(self, uhat_t, m_first: int = 0):
        g, st = self.g, self.st
        nt = self.m_last - m_first + 1
        tshape = (g.J[0], g.J1l, g.J[2])
        T = st.c2c(uhat_t, tshape, axis=0, dir=+1, w=self.w[m_first:], nterms=nt, src_ts=0, w_ts=1)
        if nt == 1 and len(T.shape) == 3:  # single term: keep the term axis for the transpose
            T = T.reshape((1,) + tuple(T.shape))
        if g.P == 1:
            Ts = T
        else:
            # T: [nt][J0][J1l][H] -> to rank q: its planes of every term
            send = [st.contig(T[:, q * g.J0l:(q + 1) * g.J0l]) for q in range(g.P)]
            recv = self.comm.all_to_all(send)                     # from p: [nt][J0l][J1l][H]
            Ts = st.concat(recv, axis=2)                          # [nt][J0l][J1][H]
        loc = (g.J0l, g.J[1], g.J[2])
        Ts = st.c2c(Ts, loc, axis=1, dir=+1, nterms=nt, src_ts=1)
        return st.c2r(Ts, loc, m_first, self.m_last, self.dev1)

    def apply(self, u_slab, m_first: int = 0):
        if m_first > self.m_last:  # perturbation of a constant order: exact zeros (flap.cpp:163-166)
            return u_slab * 0.0
        return self.inverse(self.forward(u_slab), m_first)


# --------------------------------------------------------------------------- device stages


class _CAI:
    """__cuda_array_interface__ view of a raw device pointer (zero copy into torch)."""

    def __init__(self, ptr: int, shape, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class DeviceStages:
    """The sm_100a stage kernels (C-ABI) on torch CUDA tensors.  Complex half-spectrum
    arrays are torch.complex128 tensors; everything runs on the fw context's stream."""

    def __init__(self, ctx):
        import torch

        from . import _capi

        self.torch = torch
        self.ctx = ctx
        self.lib = _capi.load_library()
        self.check = _capi.check
        self.stream = torch.cuda.ExternalStream(ctx.stream)
        lib = self.lib
        vp, ll = C.c_void_p, C.c_longlong
        lib.fw_stage_r2c.argtypes = [vp, C.c_int, C.POINTER(C.c_int), vp, vp, C.c_double]
        lib.fw_stage_c2c.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, vp, vp, vp, ll, ll, ll,
                                     C.c_int, C.c_double]
        lib.fw_stage_c2r_accum.argtypes = [vp, C.c_int, C.POINTER(C.c_int), vp, ll, C.c_int, C.c_int, vp, vp, vp]
        lib.fw_op_device_tables.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(C.c_int)]

    @staticmethod
    def _J(shape):
        return (C.c_int * 3)(*shape)

    def empty(self, shape, complex_=True):
        t = self.torch
        return t.empty(shape, dtype=t.complex128 if complex_ else t.float64, device="cuda")

    def contig(self, x):
        with self.torch.cuda.stream(self.stream):
            return x.contiguous()

    def concat(self, xs, axis):
        with self.torch.cuda.stream(self.stream):
            return self.torch.cat(xs, dim=axis)

    def r2c(self, x, shape):
        H = self.empty((shape[0], shape[1], shape[2] // 2 + 1))
        self.check(self.lib.fw_stage_r2c(self.ctx.handle, 3, self._J(shape), x.data_ptr(), H.data_ptr(), 1.0))
        return H

    def c2c(self, src, shape, axis, dir, w=None, nterms=1, src_ts=0, w_ts=0, scale=1.0):
        h = shape[2] // 2 + 1
        nh = shape[0] * shape[1] * h
        dst = self.empty(((nterms,) if nterms > 1 else ()) + (shape[0], shape[1], h))
        self.check(self.lib.fw_stage_c2c(self.ctx.handle, 3, self._J(shape), axis, dir, src.data_ptr(),
                                         dst.data_ptr(), w.data_ptr() if w is not None else None,
                                         nh * src_ts, nh, nh * w_ts, nterms, scale))
        return dst

    def c2c_scatter(self, src, shape, axis, dir, dst_ptrs, blk, jstride, ostride, tstride, base, w=None, nterms=1,
                    src_ts=0, w_ts=0, scale=1.0):
        """C2C along `axis` with the transpose fused into its last pass: output element j of
        line (o, in), term t -> dst_ptrs[j // blk][t*tstride + (j % blk)*jstride + o*ostride + in + base]
        (complex elements).  dst_ptrs: device addresses (peer memory or local)."""
        lib = self.lib
        h = shape[2] // 2 + 1
        nh = shape[0] * shape[1] * h
        P = C.c_void_p * len(dst_ptrs)
        lib.fw_stage_c2c_scatter.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_void_p,
                                             C.c_void_p, C.c_longlong, C.c_longlong, C.c_int, C.c_double, C.c_int,
                                             C.POINTER(C.c_void_p)] + [C.c_longlong] * 5
        self.check(lib.fw_stage_c2c_scatter(self.ctx.handle, 3, self._J(shape), axis, dir, src.data_ptr(),
                                            w.data_ptr() if w is not None else None, nh * src_ts, nh * w_ts, nterms,
                                            scale, len(dst_ptrs), P(*[C.c_void_p(int(x)) for x in dst_ptrs]),
                                            blk, jstride, ostride, tstride, base))

    def c2r(self, src, shape, m_first, m_last, dev1):
        out = self.empty(shape, complex_=False)
        nh = shape[0] * shape[1] * (shape[2] // 2 + 1)
        self.check(self.lib.fw_stage_c2r_accum(self.ctx.handle, 3, self._J(shape), src.data_ptr(),
                                               nh if m_last > m_first else 0, m_first, m_last,
                                               dev1.data_ptr() if dev1 is not None else None, out.data_ptr(),
                                               None))
        return out

    def local_tables(self, op, geo: SlabGeometry):
        """(w_local [M+1][J0][J1/P][H] real weights of this rank's spectral columns, dev1 of its
        planes, m_last).  A per-rank operator (api.build_slab_expansion: table bytes 1/P) is used
        as it is (zero-copy views); a full-grid operator is sliced (one gather)."""
        t = self.torch
        w, d1, ml = C.c_void_p(), C.c_void_p(), C.c_int()
        self.check(self.lib.fw_op_device_tables(op.handle, C.byref(w), C.byref(d1), C.byref(ml)))
        J0, J1, J2 = geo.J
        H = geo.H
        if getattr(op, "slab", None) is not None:
            if tuple(op.slab) != (geo.P, geo.rank):
                raise ValueError(f"operator tables are rank {op.slab[1]} of {op.slab[0]}, not {geo.rank} of {geo.P}")
            wl = t.as_tensor(_CAI(w.value, (op.M + 1, J0, geo.J1l, H)), device="cuda")
            dl = t.as_tensor(_CAI(d1.value, (geo.J0l, J1, J2)), device="cuda")
            return wl, dl, ml.value
        wt = t.as_tensor(_CAI(w.value, (op.M + 1, J0, J1, H)), device="cuda")
        dt = t.as_tensor(_CAI(d1.value, (J0, J1, J2)), device="cuda")
        with t.cuda.stream(self.stream):
            wl = wt[:, :, geo.cols, :].contiguous()
            dl = dt[geo.rows].contiguous()
        return wl, dl, ml.value


class FusedSlabApply:
    """Slab apply with both transposes FUSED into the C2C stages (fw_stage_c2c_scatter):
    the last pass of the local axis-1 C2C stores each output straight into the owning
    rank's [J0][J1/P][H] spectrum buffer, and the last pass of the all-terms axis-0 inverse
    stores into the owning rank's [nt][J0/P][J1][H] buffer -- peer memory over NVLink on a
    multi-GPU node, so the transpose overlaps the FFT instead of following it as a separate
    all-to-all.  Between the two halves of each transpose the ranks only synchronise
    (``peers.barrier()``: every rank's stores are complete).

    peers: ``T_ptrs`` / ``Ts_ptrs`` (device addresses of every rank's receive buffers, valid
    on this device), ``T(rank)`` / ``Ts(rank)`` (this rank's buffers as tensors), ``barrier()``.
    """

    def __init__(self, geo: SlabGeometry, stages, peers, w_local, dev1_local, m_last: int):
        self.g, self.st, self.peers = geo, stages, peers
        self.w, self.dev1, self.m_last = w_local, dev1_local, m_last

    # the three phases (separated by peers.barrier(); a single-process test interleaves the
    # phases of several virtual ranks)
    def phase_forward(self, u_slab):
        g, st, pe = self.g, self.st, self.peers
        J0, J1, J2 = g.J
        loc = (g.J0l, J1, J2)
        Y = st.r2c(u_slab, loc)  # R2C (axis 2), then C2C (axis 1) + transpose into every rank's T
        st.c2c_scatter(Y, loc, 1, -1, pe.T_ptrs, blk=g.J1l, jstride=g.H, ostride=g.J1l * g.H, tstride=0,
                       base=g.rank * g.J0l * g.J1l * g.H)

    def forward_spectrum(self):
        """This rank's columns of the forward spectrum (after phase_forward and a barrier)."""
        g, st, pe = self.g, self.st, self.peers
        return st.c2c(pe.T(g.rank), (g.J[0], g.J1l, g.J[2]), axis=0, dir=-1, scale=1.0 / g.N)

    def phase_inverse(self, m_first: int = 0, uhat=None):
        g, st, pe = self.g, self.st, self.peers
        J0, J1, J2 = g.J
        tshape = (J0, g.J1l, J2)
        if uhat is None:
            uhat = self.forward_spectrum()
        nt = self.m_last - m_first + 1
        # all terms: axis-0 C2C (x w_m) + transpose into every rank's Ts[nt][J0l][J1][H]
        st.c2c_scatter(uhat, tshape, 0, +1, pe.Ts_ptrs, blk=g.J0l, jstride=J1 * g.H, ostride=0,
                       tstride=g.J0l * J1 * g.H, base=g.rank * g.J1l * g.H, w=self.w[m_first:], nterms=nt,
                       src_ts=0, w_ts=1)

    def phase_finish(self, m_first: int = 0):
        g, st, pe = self.g, self.st, self.peers
        loc = (g.J0l, g.J[1], g.J[2])
        nt = self.m_last - m_first + 1
        Ts = st.c2c(pe.Ts(g.rank), loc, axis=1, dir=+1, nterms=nt, src_ts=1)
        return st.c2r(Ts, loc, m_first, self.m_last, self.dev1)

    def apply(self, u_slab, m_first: int = 0):
        if m_first > self.m_last:  # perturbation of a constant order: exact zeros (flap.cpp:163-166)
            return u_slab * 0.0
        self.phase_forward(u_slab)
        self.peers.barrier()
        self.phase_inverse(m_first)
        self.peers.barrier()
        return self.phase_finish(m_first)


class SlabSeismicStepper:
    """``SeismicStepper`` (seismic.hpp:36-46, seismic.cpp:85-142) on a slab-decomposed 3D
    grid: every rank owns planes [r J0/P, (r+1) J0/P) of the wavefields and only its slab of the
    two operators' tables (build_slab_expansion: table bytes fall as 1/P).  Per step one forward
    transform (fused transpose) shared by the two operators (orders 1+gamma and 1/2+gamma), their
    all-terms inverses (fused transposes into per-operator buffers) and the fused update.

    State: three wavefield levels and two L2prev levels rotate with the level counter (as the
    single-GPU stepper); the update of a blown-up step mins the step into EVERY rank's flag (peer
    memory), so after the next barrier all ranks freeze their later updates and the levels before
    the offending step survive.  The host reads the flag once per ``advance`` (no per-step
    collective or device-to-host read) and rewinds to the pre-step state (seismic.cpp:124-129).

    grid: the global ``Grid``; gamma, c0, phi, psi: global numpy fields (every rank passes the
    same arrays; only its slab is uploaded); peers_factory(op_index, geo, nt_max, ctx) -> peers
    (IpcPeers across processes; shared LocalPeers for virtual ranks in one process; peers of
    operator 0 also carry the blow-up flags).
    With construct=False the caller runs the constructor's three applies itself and calls
    start() (tests interleave virtual ranks that way)."""

    def __init__(self, grid, gamma, c0, omega0, M, phi, psi, tau, geo: SlabGeometry, ctx, peers_factory,
                 blowup_factor: float = 1e8, construct: bool = True):
        import torch

        from . import api
        from ._capi import check, load_library

        self.torch, self.lib, self._chk = torch, load_library(), check
        self.g, self.ctx, self.tau = geo, ctx, float(tau)
        rows = geo.rows
        J = tuple(geo.J)
        gamma, c0, phi, psi = (np.array(np.broadcast_to(np.asarray(a, dtype=np.float64), J))
                               for a in (gamma, c0, phi, psi))
        # medium coefficients of this slab (derive_medium, glibc, as the single-GPU stepper)
        self.nloc = n = geo.J0l * J[1] * J[2]
        co, eta, tc = (np.empty(n) for _ in range(3))
        lib = self.lib
        dp = C.POINTER(C.c_double)
        lib.fw_medium_coefficients.argtypes = [C.c_longlong, dp, dp, C.c_double, dp, dp, dp]
        g_loc, c0_loc = np.ascontiguousarray(gamma[rows]), np.ascontiguousarray(c0[rows])
        check(lib.fw_medium_coefficients(n, g_loc.ctypes.data_as(dp), c0_loc.ctypes.data_as(dp), float(omega0),
                                         co.ctypes.data_as(dp), eta.ctypes.data_as(dp), tc.ctypes.data_as(dp)))
        self._dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        self.c, self.eta, self.tc = self._dev(co), self._dev(eta), self._dev(tc)
        # the two operators: this rank's slab of their tables only
        self.stages = DeviceStages(ctx)
        self.ops = [api.build_slab_expansion(api.OrderField(grid, 1.0 + gamma), M, geo.P, geo.rank, ctx=ctx),
                    api.build_slab_expansion(api.OrderField(grid, 0.5 + gamma), M, geo.P, geo.rank, ctx=ctx)]
        self.table_bytes = sum(op.device_bytes for op in self.ops)
        self.apps = []
        for k, op in enumerate(self.ops):
            wl, dl, ml = self.stages.local_tables(op, geo)
            self.apps.append(FusedSlabApply(geo, self.stages, peers_factory(k, geo, ml + 1, ctx), wl, dl, ml))
        self.peers = self.apps[0].peers
        self.flag = self.peers.flag(geo.rank)
        self._pf = (C.c_void_p * len(self.peers.flag_ptrs))(*[C.c_void_p(int(x)) for x in self.peers.flag_ptrs])
        self.thr = blowup_factor * max(float(np.max(np.abs(phi))), 1e-300)  # seismic.cpp:93
        lib.fw_stage_seis_start.argtypes = [C.c_void_p, C.c_longlong, C.c_double] + [C.c_void_p] * 8
        self.ub = [torch.empty(geo.J0l * J[1] * J[2], dtype=torch.float64, device="cuda").reshape(geo.J0l, J[1], J[2])
                   for _ in range(3)]
        self.ab = [torch.empty_like(self.ub[0]) for _ in range(2)]
        self.phi_l, self.psi_l = self._dev(phi[rows]), self._dev(psi[rows])
        torch.cuda.synchronize()  # the uploads ran on torch's stream; the stepper works on the context's
        if construct:  # seismic.cpp:85-109 (one process per rank)
            self.start(self.apps[0].apply(self.phi_l), self.apps[1].apply(self.psi_l), self.apps[1].apply(self.phi_l))

    # levels: cur = ub[L % 3], prev = ub[(L + 2) % 3], next = ub[(L + 1) % 3]; L2prev = ab[(L + 1) % 2],
    # the step's new L2prev = ab[L % 2]
    @property
    def cur(self):
        return self.ub[self.lvl % 3]

    @property
    def prev(self):
        return self.ub[(self.lvl + 2) % 3]

    @property
    def l2prev(self):
        return self.ab[(self.lvl + 1) % 2]

    def start(self, l1phi, l2psi, l2phi):
        """cur = phi + tau psi + tau^2/2 c^2 (eta L1phi + tau_c L2psi), prev = phi, L2prev = L2phi, n = 1."""
        st = self.stages.stream
        self.lvl, self.n = 1, 1
        with self.torch.cuda.stream(st):
            self.prev.copy_(self.phi_l)
            self.l2prev.copy_(l2phi)
        self._chk(self.lib.fw_stage_seis_start(self.ctx.handle, self.nloc, self.tau, self.phi_l.data_ptr(),
                                                self.psi_l.data_ptr(), self.c.data_ptr(), self.eta.data_ptr(),
                                                self.tc.data_ptr(), l1phi.data_ptr(), l2psi.data_ptr(),
                                                self.cur.data_ptr()))

    # ---- one step in three phases (peers.barrier() between them; step() does it all) ----
    def phase_forward(self):
        self.apps[0].phase_forward(self.cur)  # shared forward transform (into operator 0's buffers)

    def phase_inverse(self):
        uhat = self.apps[0].forward_spectrum()
        self.apps[0].phase_inverse(0, uhat)
        self.apps[1].phase_inverse(0, uhat)

    def phase_update(self):
        """The update (seismic.cpp:116-129) into the next level; advances n and the level whether or not
        the step blew up (check() rewinds)."""
        l1, l2 = self.apps[0].phase_finish(0), self.apps[1].phase_finish(0)
        nxt, l2o = self.ub[(self.lvl + 1) % 3], self.ab[self.lvl % 2]
        self._chk(self.lib.fw_stage_seis_update_peers(
            self.ctx.handle, self.nloc, self.tau, self.cur.data_ptr(), self.prev.data_ptr(), self.l2prev.data_ptr(),
            l1.data_ptr(), l2.data_ptr(), self.c.data_ptr(), self.eta.data_ptr(), self.tc.data_ptr(), nxt.data_ptr(),
            l2o.data_ptr(), self.thr, self.n + 1, self.flag.data_ptr(), len(self.peers.flag_ptrs), self._pf))
        self.lvl += 1
        self.n += 1

    def blown(self):
        """The offending step agreed by every rank, or None.  The flag is written on the context's
        (non-blocking) stream and by the peers' updates: call after a barrier (check() does)."""
        self.ctx.sync()
        v = int(self.flag.item())
        return None if v == 0x7FFFFFFF else v

    def check(self):
        """Once per advance: after a barrier every rank's flag holds the earliest offending step over
        all ranks; rewind to the state before it and raise BlowupDetected (seismic.cpp:124-129)."""
        from ._capi import BlowupDetected

        self.peers.barrier()
        bad = self.blown()
        if bad is None:
            return
        self.lvl -= self.n - bad + 1  # the levels before the offending step (later updates were frozen)
        self.n = bad
        self.peers.barrier()  # every rank has read the flag before any resets it
        with self.torch.cuda.stream(self.stages.stream):  # ordered with the context's kernels
            self.flag.fill_(0x7FFFFFFF)
        self.ctx.sync()
        raise BlowupDetected(f"sup|u| > {self.thr:g} at step {bad}")

    def step_nocheck(self):
        self.phase_forward()
        self.peers.barrier()
        self.phase_inverse()
        self.peers.barrier()
        self.phase_update()

    def step(self):
        self.advance(1)

    def advance(self, steps: int):
        for _ in range(int(steps)):
            self.step_nocheck()
        self.check()

    def state(self):
        """(cur, prev, L2prev) of this rank's slab (torch CUDA tensors) and n."""
        return self.cur, self.prev, self.l2prev, self.n


class LocalPeers:
    """Receive buffers of P virtual ranks on ONE device (tests / single-GPU use of the fused
    path): the pointer tables address local tensors; barrier() is a stream sync.  One blow-up
    flag per virtual rank (flag(r), flag_ptrs)."""

    def __init__(self, geo: SlabGeometry, nt_max: int, ctx):
        import torch

        J0, J1, _ = geo.J
        self.ctx = ctx
        self._T = [torch.empty((J0, geo.J1l, geo.H), dtype=torch.complex128, device="cuda") for _ in range(geo.P)]
        self._Ts = [torch.empty((nt_max, geo.J0l, J1, geo.H), dtype=torch.complex128, device="cuda")
                    for _ in range(geo.P)]
        self._flags = [torch.full((1,), 0x7FFFFFFF, dtype=torch.int32, device="cuda") for _ in range(geo.P)]
        self.T_ptrs = [t.data_ptr() for t in self._T]
        self.Ts_ptrs = [t.data_ptr() for t in self._Ts]
        self.flag_ptrs = [f.data_ptr() for f in self._flags]
        torch.cuda.synchronize()  # torch filled the flags on its stream; the context's kernels use its own

    def T(self, r):
        return self._T[r]

    def Ts(self, r):
        return self._Ts[r]

    def flag(self, r):
        return self._flags[r]

    def barrier(self):
        self.ctx.sync()


class IpcPeers(LocalPeers):
    """Receive buffers of the P ranks of a torch.distributed job on one node: each rank
    allocates its own with fw_ipc_alloc (plain device allocations: a CUDA IPC handle maps the
    allocation BASE, so a buffer inside a caching allocator's block would receive peer stores at
    the wrong address), exports the handles and maps the others' (peer memory over NVLink);
    barrier() = device sync + process-group barrier."""

    def __init__(self, geo: SlabGeometry, nt_max: int, ctx):
        import torch
        import torch.distributed as dist

        from . import _capi

        J0, J1, _ = geo.J
        self.ctx, self.dist, self.torch = ctx, dist, torch
        lib, check = _capi.load_library(), _capi.check
        self._lib = lib
        lib.fw_ipc_handle.argtypes = [C.c_void_p, C.c_char_p]
        lib.fw_ipc_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.fw_ipc_close.argtypes = [C.c_void_p]
        shapes = {"T": ((J0, geo.J1l, geo.H), "<c16", 16), "Ts": ((nt_max, geo.J0l, J1, geo.H), "<c16", 16),
                  "flag": ((1,), "<i4", 4)}
        self._own, self._alloc = {}, []
        for key, (shape, typestr, esize) in shapes.items():
            ptr = C.c_void_p()
            check(lib.fw_ipc_alloc(ctx.handle, max(256, int(np.prod(shape)) * esize), C.byref(ptr)))
            self._alloc.append(ptr.value)
            self._own[key] = torch.as_tensor(_CAI(ptr.value, shape, typestr), device="cuda")
        self._own["flag"].fill_(0x7FFFFFFF)
        torch.cuda.synchronize()  # the fill ran on torch's stream, the context's kernels run on its own
        handles = []
        for key in ("T", "Ts", "flag"):
            hbuf = C.create_string_buffer(64)
            check(lib.fw_ipc_handle(C.c_void_p(self._own[key].data_ptr()), hbuf))
            handles.append(hbuf.raw)
        allh = [None] * geo.P
        dist.all_gather_object(allh, handles)
        _debug(f"rank {geo.rank}: IPC handles exchanged")
        self.T_ptrs, self.Ts_ptrs, self.flag_ptrs, self._opened = [], [], [], []
        for r, hs in enumerate(allh):
            for key, hnd, lst in zip(("T", "Ts", "flag"), hs, (self.T_ptrs, self.Ts_ptrs, self.flag_ptrs)):
                if r == geo.rank:
                    lst.append(self._own[key].data_ptr())
                    continue
                p = C.c_void_p()
                check(lib.fw_ipc_open(C.create_string_buffer(hnd, 64), C.byref(p)))
                self._opened.append(p.value)
                lst.append(p.value)
        self.rank = geo.rank
        _debug(f"rank {geo.rank}: peer buffers mapped")
        ctx.sync()
        dist.barrier()

    def T(self, r):
        assert r == self.rank
        return self._own["T"]

    def Ts(self, r):
        assert r == self.rank
        return self._own["Ts"]

    def flag(self, r):
        assert r == self.rank
        return self._own["flag"]

    def barrier(self):
        self.ctx.sync()
        self.dist.barrier()

    def close(self):
        """Unmap the peers' buffers, then free this rank's (after a barrier: no peer still writes)."""
        self.barrier()
        for p in self._opened:
            self._lib.fw_ipc_close(C.c_void_p(p))
        self._opened = []
        self.barrier()
        for p in self._alloc:
            self._lib.fw_ipc_free(self.ctx.handle, C.c_void_p(p))
        self._alloc = []


def _debug(msg):
    import os
    import sys

    if os.environ.get("FW_SLAB_DEBUG") == "1":
        print(msg, file=sys.stderr, flush=True)


class TorchComm:
    """all-to-all of equal-shape blocks over the default torch.distributed group."""

    def __init__(self, stream=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.stream = torch, dist, stream

    def all_to_all(self, blocks):
        t = self.torch
        ctx = t.cuda.stream(self.stream) if self.stream is not None else _null()
        with ctx:
            send = t.stack([b.reshape(-1) for b in blocks])
            recv = t.empty_like(send)
            if send.is_complex():
                self.dist.all_to_all_single(t.view_as_real(recv), t.view_as_real(send))
            else:
                self.dist.all_to_all_single(recv, send)
            return [recv[p].reshape(blocks[0].shape) for p in range(len(blocks))]


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def slab_apply_device(op, u_slab, geo: SlabGeometry, ctx, comm: Optional[object] = None, m_first: int = 0):
    """One distributed apply on the device: u_slab (torch CUDA float64 [J0/P][J1][J2])."""
    st = DeviceStages(ctx)
    wl, dl, ml = st.local_tables(op, geo)
    if comm is None:
        comm = TorchComm(st.stream) if geo.P > 1 else _SelfComm()
    return SlabApply(geo, st, comm, wl, dl, ml).apply(u_slab, m_first)


class _SelfComm:
    def all_to_all(self, blocks):
        return list(blocks)


def slab_of(a: np.ndarray, geo: SlabGeometry) -> np.ndarray:
    return np.ascontiguousarray(a[geo.rows])
