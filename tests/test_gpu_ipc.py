"""The fused-IPC slab path across PROCESSES: two ranks of a torch.distributed
job (gloo host group) on the one B200 of this run, every transpose a store into the peer's receive
buffer through CUDA IPC (IpcPeers: buffers from fw_ipc_alloc, handles exchanged, peer mappings),
host barriers between the phases (no kernel waits on another rank's kernel, so two processes on one
GPU are safe), blow-up flags shared through peer memory.  Results: bitwise equal to the single-GPU
SeismicStepper after 4 steps, per-rank table bytes = 1/2 of the full operator's; a blown-up run
rewinds every rank to the single-GPU stepper's pre-step state."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _case():
    J, lo, hi = (256, 256, 8), (-4.0, -4.0, -1.0), (4.0, 4.0, 1.0)
    x = [lo[a] + (hi[a] - lo[a]) * np.arange(J[a]) / J[a] for a in range(3)]
    X, Y, Z = np.meshgrid(*x, indexing="ij")
    gamma = 0.02 + 0.015 * np.sin(X) * np.cos(0.5 * Y)
    phi = np.exp(-(X**2 + Y**2 + Z**2) / 0.5)
    return J, lo, hi, gamma, phi


def _worker(rank, world, port, tau, factor, steps, q):
    try:
        _work(rank, world, port, tau, factor, steps, q)
    except BaseException as e:  # report instead of leaving the parent waiting
        import traceback

        q.put((rank, -1, "worker failed: " + "".join(traceback.format_exception(e))[-2000:], 0, None, None, None))
        os._exit(1)


def _work(rank, world, port, tau, factor, steps, q):
    import torch
    import torch.distributed as dist

    import paper_2311_13049_b200 as fw
    from paper_2311_13049_b200.slab import IpcPeers, SlabGeometry, SlabSeismicStepper

    import sys

    def say(msg):
        print(f"[rank {rank}] {msg}", file=sys.stderr, flush=True)

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    say("process group up")
    torch.cuda.set_device(0)
    ctx = fw.Context(0)
    J, lo, hi, gamma, phi = _case()
    g = fw.Grid(list(zip(lo, hi)), list(J))
    geo = SlabGeometry(J, world, rank)
    st = SlabSeismicStepper(g, gamma, np.ones(J), 1.0, 6, phi, np.zeros(J), tau, geo, ctx,
                            lambda k, geo_, nt, ctx_: IpcPeers(geo_, nt, ctx_), blowup_factor=factor)
    say(f"stepper built (table bytes {st.table_bytes})")
    err = None
    try:
        st.advance(steps)
    except fw.BlowupDetected as e:
        err = str(e)
    say(f"advanced: n = {st.n}, {err}")
    cur, prev, ap, n = st.state()
    q.put((rank, n, err, st.table_bytes, cur.cpu().numpy(), prev.cpu().numpy(), ap.cpu().numpy()))
    for a in st.apps:
        a.peers.close()
    dist.barrier()
    dist.destroy_process_group()
    os._exit(0)


def _run(world, tau, factor, steps):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tau, factor, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda r: r[0])
    for r in res:
        assert r[1] >= 0, r[2]
    for p in procs:
        p.join(timeout=120)
    return res


def _single(tau, factor, steps):
    import paper_2311_13049_b200 as fw

    J, lo, hi, gamma, phi = _case()
    g = fw.Grid(list(zip(lo, hi)), list(J))
    ref = fw.SeismicStepper(fw.build_medium(g, gamma, np.ones(J), 1.0, 6), phi, np.zeros(J), tau,
                            blowup_factor=factor)
    full_bytes = sum(i.device_bytes for i in ref.operators())
    exc = None
    try:
        ref.advance(steps)
    except fw.BlowupDetected as e:
        exc = e
    return ref, exc, full_bytes


def test_ipc_slab_two_processes_bitwise():
    res = _run(2, 1e-3, 1e8, 4)
    ref, exc, full_bytes = _single(1e-3, 1e8, 4)
    assert exc is None and all(r[2] is None for r in res)
    cur_r, prev_r, ap_r, n_r = ref.state()
    assert all(r[1] == n_r for r in res)
    for i, want in zip((4, 5, 6), (cur_r, prev_r, ap_r)):
        assert np.array_equal(np.concatenate([r[i] for r in res]), want)
    # per-rank resident tables: half of each operator's w (spectral columns) and dev1 (planes)
    for r in res:
        print(f"rank {r[0]}: table bytes {r[3]} (single-device operators: {full_bytes})")
        assert r[3] * 2 <= full_bytes + 1024


def test_ipc_slab_two_processes_blowup():
    # probe the single-GPU growth to place the threshold between steps 4 and 5 (as the virtual-rank test)
    import paper_2311_13049_b200 as fw

    J, lo, hi, gamma, phi = _case()
    g = fw.Grid(list(zip(lo, hi)), list(J))
    probe = fw.SeismicStepper(fw.build_medium(g, gamma, np.ones(J), 1.0, 6), phi, np.zeros(J), 0.2,
                              blowup_factor=1e300)
    sups = []
    for _ in range(4):
        probe.step()
        sups.append(np.abs(probe.current()).max())
    factor = np.sqrt(max(max(sups[:3]), 1.0) * sups[3]) / np.abs(phi).max()
    ref, exc, _ = _single(0.2, factor, 6)
    assert exc is not None and ref.n() == 5
    res = _run(2, 0.2, factor, 6)
    assert all(r[1] == 5 and r[2] is not None for r in res)
    cur_r, prev_r, ap_r, _ = ref.state()
    for i, want in zip((4, 5, 6), (cur_r, prev_r, ap_r)):
        assert np.array_equal(np.concatenate([r[i] for r in res]), want)


@pytest.mark.parametrize("blowup", [False, True])
def test_c_abi_slab_stepper_p1_vs_single_gpu(blowup):
    """The C++ slab stepper of the C-ABI (fw_slab_seis_*; P = 1 on this one-GPU run: the same stage,
    scatter, update and flag code as P > 1, the transposes into the own buffers): bitwise equal to
    the single-GPU SeismicStepper, including a blow-up rewind."""
    import paper_2311_13049_b200 as fw

    J, lo, hi, gamma, phi = _case()
    g = fw.Grid(list(zip(lo, hi)), list(J))
    tau, factor, steps = (1e-3, 1e8, 5) if not blowup else (0.2, 1.0, 6)
    if blowup:  # threshold between the sups of steps 4 and 5 (see the IPC blow-up test)
        probe = fw.SeismicStepper(fw.build_medium(g, gamma, np.ones(J), 1.0, 6), phi, np.zeros(J), tau,
                                  blowup_factor=1e300)
        sups = []
        for _ in range(4):
            probe.step()
            sups.append(np.abs(probe.current()).max())
        factor = np.sqrt(max(max(sups[:3]), 1.0) * sups[3]) / np.abs(phi).max()
    ref = fw.SeismicStepper(fw.build_medium(g, gamma, np.ones(J), 1.0, 6), phi, np.zeros(J), tau, blowup_factor=factor)
    st = fw.SlabSeismicStepperC(g, gamma, np.ones(J), 1.0, 6, phi, np.zeros(J), tau, blowup_factor=factor)
    e1 = e2 = None
    try:
        ref.advance(steps)
    except fw.BlowupDetected as e:
        e1 = e
    try:
        st.advance(steps)
    except fw.BlowupDetected as e:
        e2 = e
    assert (e1 is None) == (e2 is None) == (not blowup)
    cur, prev, ap, n = st.state()
    rcur, rprev, rap, rn = ref.state()
    assert n == rn
    assert np.array_equal(cur, rcur) and np.array_equal(prev, rprev) and np.array_equal(ap, rap)
    assert st.table_bytes > 0
