"""Small driver for ncu: C3 grid (512^2) with a short window, runs the
kernel timing probe (TLM stage + column kernels) on one sweep group."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import scenario  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
group = int(sys.argv[2]) if len(sys.argv) > 2 else 0
stages = int(sys.argv[3]) if len(sys.argv) > 3 else 16
sdv.init(0)
spec = scenario.with_window(scenario.CONFIGS[cfg], steps=8, spi=8)
sc = scenario.build(spec, block_group=group)
tr = sc.problem.linearize(sc.problem.background)
s = spec.rank
ms_stage, ms_col = tr.probe_stage_kernels(s, stages)
print(f"config {cfg} group {group}: stage kernel {ms_stage*1e3:.1f} us, col kernel {ms_col*1e3:.1f} us")
