"""Sketch columns sharded over ranks, one process per GPU.

The reference's parallel unit is the column fan-out of one sketch:
randsvd_sketch (proj/src/sketch.cpp:142-160) pushes the l columns of its
Gaussian test block through apply_columns (proj/src/sketch.cpp:116-140), whose
worker threads each run whole TLM or ADJ sweeps of single columns. Here the
columns are split over ranks instead of threads: rank r owns the contiguous
slice column_shard(l, world, r) and runs its columns as one device block
(one block sweep per rank, every rank against its own copy of the same
deterministic base trajectory).

Nystrom (Algorithm 2, nystrom_sharded) has one exchange: Y = H Omega (n x l)
is all-gathered and every rank runs the stabilised assembly. RandSVD
(Algorithm 1) has two exchange steps, and these are the only collectives on
its path:
  1. Y = A Omega (m x l): each rank holds the columns of its slice; an
     all-gather assembles Y, and every rank factorises the same Y with the same
     device QR (sdv_thin_qr_dev: CholQR2 / Householder), so Q is replicated
     identically;
  2. W^T = A^T Q (n x l): each rank sweeps its slice of Q's columns; an
     all-gather assembles W^T and every rank runs the l x l tail
     (sdv_evd_from_tall_dev: QR of W^T, SVD of R), so the basis V_hat that PCG
     needs is replicated on every rank (the "all-gather of V_hat before PCG"
     of SURVEY 8(e)).
The sweeps dominate (seconds per block at C3); the all-gathers move
8 m l + 8 n l bytes (36 MB + 230 MB at C3, well under a millisecond at NVLink
bandwidth). PCG and the line search are sequential: replicas only.

Communication goes through a small `comm` object (rank, world, allgather_rows).
TorchComm uses torch.distributed (NCCL on GPUs, gloo on CPU) and is the
production path; ThreadComm runs the ranks as threads of one process (used to
exercise the sharded path on a single GPU without ranks whose kernels wait on
one another: the collectives synchronise host threads, never kernels).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from ._lib import check, lib
from .api import gaussian_matrix


def column_shard(l, world, rank):
    """Contiguous slice [lo, hi) of l columns owned by `rank` of `world`
    (the first l % world ranks own one extra column)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("column_shard: need 0 <= rank < world")
    base, extra = divmod(l, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather_rows(self, x, counts):
        """Row blocks x (counts[rank] x k) of every rank -> (sum(counts) x k) in rank order."""
        import torch

        mx = max(counts)
        pad = x.new_zeros((mx,) + tuple(x.shape[1:]))
        pad[: x.shape[0]] = x
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self._dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


class ThreadComm:
    """`world` ranks as threads of one process; allgather_rows meets at a barrier."""

    def __init__(self, world):
        self.world = world
        self._slots = [None] * world
        self._bar = threading.Barrier(world)

    def view(self, rank):
        comm = self

        class _View:
            def __init__(self):
                self.world, self.rank = comm.world, rank

            def allgather_rows(self, x, counts):
                import torch

                comm._slots[rank] = x
                comm._bar.wait()
                out = torch.cat([comm._slots[r][:c] for r, c in enumerate(counts)], dim=0)
                comm._bar.wait()  # every rank has read the slots before any rank reuses them
                return out

        return _View()


class GpuSketchOps:
    """Device operations of one rank over the C-ABI, on torch CUDA tensors
    (row-major (k, n) tensors are column-major n x k blocks)."""

    def __init__(self, traj, device=None):
        import torch

        self.torch = torch
        self.traj = traj
        self.problem = traj.problem
        self.n, self.m = self.problem.n, self.problem.m
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def _sync_in(self):
        self.torch.cuda.synchronize(self.device)  # torch-side writes visible to the library stream

    def _sync_out(self):
        self.problem.synchronize()  # library stream done before torch / NCCL read the result

    def gaussian(self, l, seed):
        return gaussian_matrix(self.n, l, seed)

    def apply(self, V):
        """Y = A V (TLM block sweep): V host (k, n) -> device (k, m)."""
        t = self.torch
        v = t.as_tensor(np.ascontiguousarray(V), dtype=t.float64, device=self.device)
        y = t.empty((v.shape[0], self.m), dtype=t.float64, device=self.device)
        if v.shape[0]:
            self._sync_in()
            check(lib().sdv_misfit_apply_block_dev(self.traj.handle, C.c_void_p(v.data_ptr()), v.shape[0],
                                                   C.c_void_p(y.data_ptr())))
            self._sync_out()
        return y

    def adjoint(self, W):
        """Z = A^T W (ADJ block sweep): device (k, m) -> device (k, n)."""
        t = self.torch
        w = W.contiguous()
        z = t.empty((w.shape[0], self.n), dtype=t.float64, device=self.device)
        if w.shape[0]:
            self._sync_in()
            check(lib().sdv_misfit_adjoint_block_dev(self.traj.handle, C.c_void_p(w.data_ptr()), w.shape[0],
                                                     C.c_void_p(z.data_ptr())))
            self._sync_out()
        return z

    def gram(self, V):
        """H V = A^T A V (TLM + ADJ block sweeps): V host (k, n) -> device (k, n)."""
        t = self.torch
        v = t.as_tensor(np.ascontiguousarray(V), dtype=t.float64, device=self.device)
        hv = t.empty_like(v)
        if v.shape[0]:
            self._sync_in()
            check(lib().sdv_gram_apply_block_dev(self.traj.handle, C.c_void_p(v.data_ptr()), v.shape[0],
                                                 C.c_void_p(hv.data_ptr())))
            self._sync_out()
        return hv

    def nystrom_assemble(self, omega, Y):
        """nystrom_assemble (proj/src/sketch.cpp:162-200) of host Omega (l, n) and device Y (l, n)."""
        t = self.torch
        l, n = Y.shape
        om = t.as_tensor(np.ascontiguousarray(omega), dtype=t.float64, device=self.device)
        eig = np.empty(l)
        basis = t.empty((l, n), dtype=t.float64, device=self.device)
        self._sync_in()
        check(lib().sdv_nystrom_assemble_dev(self.problem.handle, n, l, C.c_void_p(om.data_ptr()),
                                             C.c_void_p(Y.data_ptr()), C.c_void_p(basis.data_ptr()),
                                             eig.ctypes.data_as(C.POINTER(C.c_double))))
        return eig, basis

    def qr_(self, Y):
        """In-place device thin QR (the sketches' QR, proj/src/linalg.cpp:108-134): Y (l, m) -> Q."""
        l, m = Y.shape
        r = np.empty((l, l))
        nd = C.c_int()
        self._sync_in()
        check(lib().sdv_thin_qr_dev(self.problem.handle, m, l, C.c_void_p(Y.data_ptr()),
                                    r.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nd)))
        return Y

    def evd_from_tall(self, Wt):
        """evd_from_gram_factor (proj/src/sketch.cpp:27-33) of W^T (l, n): eigenvalues, basis (l, n)."""
        t = self.torch
        l, n = Wt.shape
        eig = np.empty(l)
        basis = t.empty((l, n), dtype=t.float64, device=self.device)
        self._sync_in()
        check(lib().sdv_evd_from_tall_dev(self.problem.handle, n, l, C.c_void_p(Wt.data_ptr()), 0.0, 0,
                                          C.c_void_p(basis.data_ptr()), eig.ctypes.data_as(C.POINTER(C.c_double))))
        return eig, basis


def randsvd_sharded(ops, rank, seed, comm=None):
    """randsvd_sketch(A, rank, seed) (proj/src/sketch.cpp:142-160) with Omega's
    columns sharded over comm's ranks. Returns (eig, basis, counts); every
    rank returns the same eigenvalues and basis. counts = {tlm, adj,
    final_rank} of the whole sketch (as the single-process sketch reports)
    plus this rank's column slice."""
    if comm is None:
        comm = TorchComm()
    if rank < 1 or rank > min(ops.m, ops.n):
        raise ValueError("randsvd_sketch: need 1 <= rank <= min(m, n)")
    counts = [column_shard(rank, comm.world, r) for r in range(comm.world)]
    widths = [hi - lo for lo, hi in counts]
    lo, hi = counts[comm.rank]
    omega = ops.gaussian(rank, seed)  # bit-exact host draws, identical on every rank
    y_local = ops.apply(omega[lo:hi])  # this rank's TLM sweeps
    y = comm.allgather_rows(y_local, widths)  # exchange 1: Y (m x l)
    q = ops.qr_(y)  # replicated QR
    wt_local = ops.adjoint(q[lo:hi])  # this rank's ADJ sweeps
    wt = comm.allgather_rows(wt_local, widths)  # exchange 2: W^T (n x l)
    eig, basis = ops.evd_from_tall(wt)  # replicated tail -> V_hat on every rank
    return eig, basis, {"tlm": rank, "adj": rank, "final_rank": rank, "columns": (lo, hi)}


def nystrom_sharded(ops, rank, seed, comm=None):
    """nystrom_sketch(H, rank, seed) (proj/src/sketch.cpp:202-220) with Omega's
    columns sharded over comm's ranks: each rank applies H = A^T A to its
    columns (one TLM + ADJ block sweep), Y = H Omega is all-gathered, and every
    rank runs the same stabilised assembly (replicated basis)."""
    if comm is None:
        comm = TorchComm()
    if rank < 1 or rank > ops.n:
        raise ValueError("nystrom_sketch: need 1 <= rank <= n")
    counts = [column_shard(rank, comm.world, r) for r in range(comm.world)]
    widths = [hi - lo for lo, hi in counts]
    lo, hi = counts[comm.rank]
    omega = ops.gaussian(rank, seed)
    y = comm.allgather_rows(ops.gram(omega[lo:hi]), widths)  # the one exchange: Y (n x l)
    eig, basis = ops.nystrom_assemble(omega, y)
    return eig, basis, {"tlm": rank, "adj": rank, "final_rank": rank, "columns": (lo, hi)}


def run_threads(world, fn):
    """Run fn(comm_view) on `world` threads (ThreadComm) and return the per-rank results."""
    comm = ThreadComm(world)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            out[r] = fn(comm.view(r))
        except BaseException as e:  # surfaced below
            err[r] = e
            comm._bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out
