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
        """(w_local [M+1][J0][J1/P][H] complex-layout-compatible real weights, dev1 slab, m_last)
        sliced from the operator's resident device tables (zero-copy views + one gather)."""
        t = self.torch
        w, d1, ml = C.c_void_p(), C.c_void_p(), C.c_int()
        self.check(self.lib.fw_op_device_tables(op.handle, C.byref(w), C.byref(d1), C.byref(ml)))
        J0, J1, J2 = geo.J
        H = geo.H
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
    grid: every rank owns planes [r J0/P, (r+1) J0/P) of the wavefields.  Per step one
    forward transform (fused transpose) shared by the two operators (orders 1+gamma and
    1/2+gamma), their all-terms inverses (fused transposes into per-operator buffers), and
    the fused update; the blow-up flag is combined over the ranks every step, and on a
    blow-up every rank keeps its pre-step state (reference semantics).

    grid: the global ``Grid``; gamma, c0, phi, psi: global numpy fields (every rank passes the
    same arrays; only its slab is uploaded); peers_factory(op_index, geo, nt_max, ctx) -> peers
    (IpcPeers across processes; shared LocalPeers for virtual ranks in one process).
    With construct=False the caller runs the constructor's three applies itself and calls
    start() (tests interleave virtual ranks that way)."""

    def __init__(self, grid, gamma, c0, omega0, M, phi, psi, tau, geo: SlabGeometry, ctx, peers_factory,
                 blowup_factor: float = 1e8, flag_reduce=None, construct: bool = True):
        import torch

        from . import api
        from ._capi import check, load_library

        self.torch, self.lib, self.check = torch, load_library(), check
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
        # the two operators (full tables on every rank, sliced to the slab)
        self.stages = DeviceStages(ctx)
        self.ops = [api.build_expansion(api.OrderField(grid, 1.0 + gamma), M, ctx=ctx),
                    api.build_expansion(api.OrderField(grid, 0.5 + gamma), M, ctx=ctx)]
        self.apps = []
        for k, op in enumerate(self.ops):
            wl, dl, ml = self.stages.local_tables(op, geo)
            self.apps.append(FusedSlabApply(geo, self.stages, peers_factory(k, geo, ml + 1, ctx), wl, dl, ml))
        self.peers = self.apps[0].peers
        self.flag = torch.full((1,), 0x7FFFFFFF, dtype=torch.int32, device="cuda")
        self.flag_reduce = flag_reduce
        self.thr = blowup_factor * max(float(np.max(np.abs(phi))), 1e-300)  # seismic.cpp:93
        lib.fw_stage_seis_start.argtypes = [C.c_void_p, C.c_longlong, C.c_double] + [C.c_void_p] * 8
        lib.fw_stage_seis_update.argtypes = ([C.c_void_p, C.c_longlong, C.c_double] + [C.c_void_p] * 9
                                             + [C.c_double, C.c_int, C.c_void_p])
        self.phi_l, self.psi_l = self._dev(phi[rows]), self._dev(psi[rows])
        if construct:  # seismic.cpp:85-109 (one process per rank)
            self.start(self.apps[0].apply(self.phi_l), self.apps[1].apply(self.psi_l), self.apps[1].apply(self.phi_l))

    def start(self, l1phi, l2psi, l2phi):
        """cur = phi + tau psi + tau^2/2 c^2 (eta L1phi + tau_c L2psi), prev = phi, L2prev = L2phi, n = 1."""
        cur = self.torch.empty_like(self.phi_l)
        self.check(self.lib.fw_stage_seis_start(self.ctx.handle, self.nloc, self.tau, self.phi_l.data_ptr(),
                                                self.psi_l.data_ptr(), self.c.data_ptr(), self.eta.data_ptr(),
                                                self.tc.data_ptr(), l1phi.data_ptr(), l2psi.data_ptr(),
                                                cur.data_ptr()))
        self.prev, self.cur, self.l2prev, self.n = self.phi_l, cur, l2phi, 1

    # ---- one step in three phases (peers.barrier() between them; step() does it all) ----
    def phase_forward(self):
        self.apps[0].phase_forward(self.cur)  # shared forward transform (into operator 0's buffers)

    def phase_inverse(self):
        uhat = self.apps[0].forward_spectrum()
        self.apps[0].phase_inverse(0, uhat)
        self.apps[1].phase_inverse(0, uhat)

    def phase_update(self):
        l1, l2 = self.apps[0].phase_finish(0), self.apps[1].phase_finish(0)
        self._next = self.torch.empty_like(self.cur)
        self._l2 = l2
        self.check(self.lib.fw_stage_seis_update(self.ctx.handle, self.nloc, self.tau, self.cur.data_ptr(),
                                                 self.prev.data_ptr(), self.l2prev.data_ptr(), l1.data_ptr(),
                                                 l2.data_ptr(), self.c.data_ptr(), self.eta.data_ptr(),
                                                 self.tc.data_ptr(), self._next.data_ptr(), self.thr, self.n + 1,
                                                 self.flag.data_ptr()))

    def blown(self):
        """The offending step over all ranks (flag_reduce = a min all-reduce), or None.
        fw_stage_seis_update wrote the flag on the context's (non-blocking) stream: wait for
        it before torch reads the flag on its own stream."""
        self.ctx.sync()
        f = self.flag.clone()
        if self.flag_reduce is not None:
            f = self.flag_reduce(f)
        v = int(f.item())
        return None if v == 0x7FFFFFFF else v

    def commit(self):
        self.prev, self.cur, self.l2prev = self.cur, self._next, self._l2
        self.n += 1

    def step(self):
        from ._capi import BlowupDetected

        self.phase_forward()
        self.peers.barrier()
        self.phase_inverse()
        self.peers.barrier()
        self.phase_update()
        bad = self.blown()
        if bad is not None:  # the state stays the pre-step one (seismic.cpp:124-129)
            raise BlowupDetected(f"sup|u| > {self.thr:g} at step {bad}")
        self.commit()

    def advance(self, steps: int):
        for _ in range(int(steps)):
            self.step()

    def state(self):
        """(cur, prev, L2prev) of this rank's slab (torch CUDA tensors) and n."""
        return self.cur, self.prev, self.l2prev, self.n


class LocalPeers:
    """Receive buffers of P virtual ranks on ONE device (tests / single-GPU use of the fused
    path): the pointer tables address local tensors; barrier() is a stream sync."""

    def __init__(self, geo: SlabGeometry, nt_max: int, ctx):
        import torch

        J0, J1, _ = geo.J
        self.ctx = ctx
        self._T = [torch.empty((J0, geo.J1l, geo.H), dtype=torch.complex128, device="cuda") for _ in range(geo.P)]
        self._Ts = [torch.empty((nt_max, geo.J0l, J1, geo.H), dtype=torch.complex128, device="cuda")
                    for _ in range(geo.P)]
        self.T_ptrs = [t.data_ptr() for t in self._T]
        self.Ts_ptrs = [t.data_ptr() for t in self._Ts]

    def T(self, r):
        return self._T[r]

    def Ts(self, r):
        return self._Ts[r]

    def barrier(self):
        self.ctx.sync()


class IpcPeers(LocalPeers):
    """Receive buffers of the P ranks of a torch.distributed job on one node: each rank
    allocates its own, exports CUDA IPC handles, and maps the others' (peer memory over
    NVLink); barrier() = device sync + process-group barrier."""

    def __init__(self, geo: SlabGeometry, nt_max: int, ctx):
        import torch
        import torch.distributed as dist

        J0, J1, _ = geo.J
        self.ctx, self.dist = ctx, dist
        self._mine_T = torch.empty((J0, geo.J1l, geo.H), dtype=torch.complex128, device="cuda")
        self._mine_Ts = torch.empty((nt_max, geo.J0l, J1, geo.H), dtype=torch.complex128, device="cuda")
        from . import _capi

        lib, check = _capi.load_library(), _capi.check
        lib.fw_ipc_handle.argtypes = [C.c_void_p, C.c_char_p]
        lib.fw_ipc_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        handles = []
        for t in (self._mine_T, self._mine_Ts):
            hbuf = C.create_string_buffer(64)
            check(lib.fw_ipc_handle(C.c_void_p(t.data_ptr()), hbuf))
            handles.append(hbuf.raw)
        allh = [None] * geo.P
        dist.all_gather_object(allh, handles)
        self.T_ptrs, self.Ts_ptrs = [], []
        for r, (hT, hTs) in enumerate(allh):
            if r == geo.rank:
                self.T_ptrs.append(self._mine_T.data_ptr())
                self.Ts_ptrs.append(self._mine_Ts.data_ptr())
                continue
            for hnd, lst in ((hT, self.T_ptrs), (hTs, self.Ts_ptrs)):
                p = C.c_void_p()
                check(lib.fw_ipc_open(C.create_string_buffer(hnd, 64), C.byref(p)))
                lst.append(p.value)
        self.rank = geo.rank

    def T(self, r):
        assert r == self.rank
        return self._mine_T

    def Ts(self, r):
        assert r == self.rank
        return self._mine_Ts

    def barrier(self):
        self.ctx.sync()
        self.dist.barrier()


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
