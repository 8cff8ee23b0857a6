"""Per-vector stage/col kernel time vs sweep group size on a config grid."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import scenario  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
groups = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [6, 9, 14, 23, 37, 55, 110]
sdv.init(0)
spec = scenario.with_window(scenario.CONFIGS[cfg], steps=8, spi=8)
for g in groups:
    sc = scenario.build(spec, block_group=g)
    tr = sc.problem.linearize(sc.problem.background)
    ms_stage, ms_col = tr.probe_stage_kernels(g, 32)
    print(f"cfg {cfg} g={g:4d}: stage {ms_stage*1e3:8.1f} us ({ms_stage*1e3/g:6.2f}/vec)  "
          f"col {ms_col*1e3:8.1f} us ({ms_col*1e3/g:6.2f}/vec)  total/vec {(ms_stage+ms_col)*1e3/g:6.2f} us", flush=True)
    del tr, sc
