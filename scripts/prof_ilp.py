"""ILP model build on the final BERT e-graph: device skeleton (tsat_ilp_build +
download) vs host row materialisation and LP export."""
import sys
import time

sys.path.insert(0, ".")
from paper_2101_01332_b200 import models  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, explore  # noqa: E402
from paper_2101_01332_b200.extract import _ilp_skeleton, build_ilp, export_lp  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402

eg, filt, rep = explore(models.MODELS["bert"](), list(default_rules()), ExploreLimits(k_multi=1))
costs = egraph_costs(eg, CostModel())
for i in range(3):
    t0 = time.perf_counter()
    sk = _ilp_skeleton(eg, filt)
    t1 = time.perf_counter()
    m = build_ilp(eg, costs, filt)
    t2 = time.perf_counter()
    nrows = len(m.rows)
    t3 = time.perf_counter()
    lp = export_lp(m)
    t4 = time.perf_counter()
print(f"nodes {eg.num_nodes} classes {len(sk['classes'])} x-vars {len(sk['nodes'])} rows {nrows} lp {len(lp)} B")
print(f"skeleton (device build + download) {1e3*(t1-t0):.2f} ms, build_ilp {1e3*(t2-t1):.2f} ms, "
      f"rows {1e3*(t3-t2):.1f} ms, export_lp {1e3*(t4-t3):.1f} ms")
