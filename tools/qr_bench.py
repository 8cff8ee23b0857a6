"""Time the sketches' thin QR on the device at the C3 sketch shapes (l = 110:
Y is m x l, m = 40960; W^T is n x l, n = 262144) and check it: CholQR2 on the
DMMA Gram (default) vs Householder (SDV_QR=householder, set before the first
call). Prints ms per QR (CUDA events), ||Q^T Q - I||_max and ||Q R - Y|| / ||Y||.

usage: python tools/qr_bench.py            (both paths, one subprocess each)
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one():
    import numpy as np
    import torch

    import paper_2401_15758_b200 as sdv
    from paper_2401_15758_b200 import api, scenario
    from paper_2401_15758_b200._lib import check, lib

    sdv.init(0)
    sc = scenario.build(scenario.with_window(scenario.CONFIGS[0], steps=10, spi=10))
    prob = sc.problem
    out = []
    for rows, l in ((40960, 110), (262144, 110), (65536, 100)):
        g = torch.Generator().manual_seed(1)
        base = torch.randn(l, rows, generator=g, dtype=torch.float64)
        base[:, :] += 0.1 * torch.randn(1, rows, generator=g, dtype=torch.float64)  # some column correlation
        ref = base.cuda()
        r = np.empty((l, l))
        nd = C.c_int()
        times = []
        for it in range(4):
            y = ref.clone()
            torch.cuda.synchronize()
            e0, e1 = api.Event(), api.Event()
            e0.record(prob)
            check(lib().sdv_thin_qr_dev(prob.handle, rows, l, C.c_void_p(y.data_ptr()),
                                        r.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nd)))
            e1.record(prob)
            times.append(e0.elapsed_ms(e1))
        q = y
        orth = (q @ q.T - torch.eye(l, device="cuda", dtype=torch.float64)).abs().max().item()
        # r holds R column-major, so as a C-order array it is R^T; y rows are Y's columns: Y^T = R^T Q^T
        resid = (torch.from_numpy(np.ascontiguousarray(r)).cuda() @ q - ref).norm().item() / ref.norm().item()
        out.append(dict(rows=rows, l=l, ms=min(times[1:]), orth=orth, resid=resid, diag_min=float(np.diag(r).min())))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        import json

        print(json.dumps(run_one()))
        sys.exit(0)
    for mode in ("cholqr2", "householder"):
        env = dict(os.environ)
        if mode == "householder":
            env["SDV_QR"] = "householder"
        else:
            env.pop("SDV_QR", None)
        res = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
        print(mode, res.stdout.strip() or res.stderr[-2000:])
