"""Short workload for one ncu capture of the round-2 kernels: the DMMA Gram of
the sketches' CholQR2 at a C3 shape (n = 262144, l = 110) and one C1 Burgers
block Gram sweep (s = 60, TMA-fed base rows)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import api, scenario  # noqa: E402
from paper_2401_15758_b200._lib import check, lib  # noqa: E402

sdv.init(0)
sc = scenario.build(1)
prob = sc.problem
tr = prob.linearize(prob.background)
y = torch.randn(110, 262144, dtype=torch.float64, device="cuda")
r = np.empty((110, 110))
nd = C.c_int()
torch.cuda.synchronize()
check(lib().sdv_thin_qr_dev(prob.handle, 262144, 110, C.c_void_p(y.data_ptr()),
                            r.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nd)))
V = api.gaussian_matrix(prob.n, 60, 3)
HV = tr.gram(V)
print("ok", float(np.abs(HV).max()))
