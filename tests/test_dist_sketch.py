"""Sharded sketch: RandSVD with Omega's columns split over
ranks, two all-gathers (Y, then W^T), replicated QR and l x l tail
(paper_2401_15758_b200/dist.py; reference: randsvd_sketch + apply_columns,
proj/src/sketch.cpp:116-160).

CPU: world size 2 over gloo, with the oracle as each rank's operator backend
(test infrastructure), against the oracle's single-process sketch — the host
logic (sharding, gather order, padding of uneven shards, replicated tail).
GPU: the device backend over the C-ABI with the ranks as threads of one
process (ThreadComm; no kernels wait on one another), against the device's
own single-process sketch and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2401_15758_b200 import dist as sdist


def test_column_shard_covers_every_column_once():
    for l in (1, 5, 30, 110):
        for world in (1, 2, 3, 4, 8):
            spans = [sdist.column_shard(l, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == l
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            widths = [hi - lo for lo, hi in spans]
            assert max(widths) - min(widths) <= 1
    with pytest.raises(ValueError):
        sdist.column_shard(10, 2, 2)


class OracleOps:
    """Oracle-backed rank operations (CPU tensors) for the host-logic test."""

    def __init__(self, otr, n, m):
        import oracle_lib

        self.o = oracle_lib
        self.otr, self.n, self.m = otr, n, m
        self.device = torch.device("cpu")

    def gaussian(self, l, seed):
        return self.o.gaussian_matrix(self.n, l, seed)

    def apply(self, V):
        return torch.from_numpy(self.otr.misfit_apply(np.ascontiguousarray(V)))

    def adjoint(self, W):
        return torch.from_numpy(self.otr.misfit_adjoint(np.ascontiguousarray(W.numpy())))

    def qr_(self, Y):
        q, _, _ = self.o.thin_qr(Y.numpy().T)
        Y.copy_(torch.from_numpy(np.ascontiguousarray(q.T)))
        return Y

    def evd_from_tall(self, Wt):
        # evd_from_gram_factor(W) = thin_svd(W): basis = V, eigenvalues = s^2 (oracle/src/sketch.cpp:19-26)
        _, s, v = self.o.thin_svd(Wt.numpy())
        return s * s, torch.from_numpy(np.ascontiguousarray(v.T))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, steps, l, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    import oracle_lib

    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        osc = oracle_lib.Scenario(cfg, steps=steps)
        otr = osc.linearize(osc.background)
        ops = OracleOps(otr, osc.n, osc.n_obs * osc.n_t)
        eig, basis, cnt = sdist.randsvd_sharded(ops, l, seed, sdist.TorchComm())
        q.put((rank, eig, basis.numpy(), cnt["columns"]))
        dist.destroy_process_group()
    except BaseException as e:  # surface the failure instead of a queue timeout
        q.put((rank, repr(e), None, None))
        raise


@pytest.mark.parametrize("cfg,steps,l", [(0, -1, 9), (2, 20, 7)])
def test_sharded_randsvd_two_ranks_gloo_equals_single_process(cfg, steps, l):
    import oracle_lib

    world, port, seed = 2, _free_port(), 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, steps, l, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    assert all(r[2] is not None for r in res), [r[1] for r in res]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    osc = oracle_lib.Scenario(cfg, steps=steps)
    eo, bo, co = osc.linearize(osc.background).sketch(0, l, seed)
    assert [r[3] for r in res] == [(0, (l + 1) // 2), ((l + 1) // 2, l)]  # uneven shards when l is odd
    for _, eig, basis, _ in res:
        assert np.array_equal(eig, eo)  # same columns, same QR, same tail: bitwise
        assert np.array_equal(np.abs(basis), np.abs(bo))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,steps,spi,l,world", [(0, -1, -1, 30, 2), (2, 20, -1, 12, 3), (3, 8, 4, 110, 2)])
def test_sharded_randsvd_threads_on_gpu(oracle, sdv, cfg, steps, spi, l, world):
    """Sharded RandSVD eigenvalues equal the single-process device sketch and
    the oracle's to <= 1e-10 (the shards run narrower blocks, so other kernel
    paths: agreement is to roundoff, not bitwise)."""
    from test_gpu_parity import eig_rel, pair

    osc, prob = pair(oracle, cfg, steps, spi)
    gtr = prob.linearize(osc.background)
    seed = oracle.mix_seed(2, 0x736b6574636800)
    eg, bg, _ = gtr.sketch(0, l, seed)
    ops = sdist.GpuSketchOps(gtr)
    outs = sdist.run_threads(world, lambda comm: sdist.randsvd_sharded(ops, l, seed, comm))
    e0, b0, c0 = outs[0]
    for e, b, c in outs[1:]:
        assert np.array_equal(e, e0) and torch.equal(b, b0)  # replicated tail: identical on every rank
    assert c0["tlm"] == l and c0["adj"] == l
    assert eig_rel(e0, eg) <= 1e-10
    b0 = b0.cpu().numpy()
    # same subspace as the single-process basis (columns agree up to sign)
    k = min(l, 10)
    assert np.allclose(np.abs(np.sum(b0[:k] * bg[:k], axis=1)), 1.0, atol=1e-8)
    if l <= 30:
        otr = osc.linearize(osc.background)
        eo, _, _ = otr.sketch(0, l, seed, workers=max(2, os.cpu_count() or 2))
        assert eig_rel(e0, eo) <= 1e-8


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,steps,spi,l,world", [(0, -1, -1, 30, 2), (2, 20, -1, 50, 2), (1, -1, -1, 60, 4)])
def test_sharded_nystrom_threads_on_gpu(oracle, sdv, cfg, steps, spi, l, world):
    """Sharded Nystrom (one all-gather of Y = H Omega, replicated assembly) vs the single-process device
    sketch (<= 1e-10) and the oracle (<= 1e-8): C0, C2's config sketch (k = 40, p = 10), C1 (k = 50, p = 10)."""
    from test_gpu_parity import eig_rel, pair

    osc, prob = pair(oracle, cfg, steps, spi)
    gtr = prob.linearize(osc.background)
    seed = oracle.mix_seed(2, 0x736b6574636800)
    eg, _, _ = gtr.sketch(1, l, seed)
    ops = sdist.GpuSketchOps(gtr)
    outs = sdist.run_threads(world, lambda comm: sdist.nystrom_sharded(ops, l, seed, comm))
    e0, b0, c0 = outs[0]
    for e, b, c in outs[1:]:
        assert np.array_equal(e, e0) and torch.equal(b, b0)
    assert c0["tlm"] == l and c0["adj"] == l
    assert eig_rel(e0, eg) <= 1e-10
    otr = osc.linearize(osc.background)
    eo, _, _ = otr.sketch(1, l, seed, workers=max(2, os.cpu_count() or 2))
    assert eig_rel(e0, eo) <= 1e-8
