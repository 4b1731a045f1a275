"""B200-native equality-saturation engine for Tensat-style tensor-graph
superoptimisation (arXiv 2101.01332).

Host modules keep the reference ``tensorsat`` API (explore / saturate /
greedy_extract / egraph_costs / run_optimize and the graph, rule and cost
formats); the e-graph itself lives on the GPU inside ``libtsat.so``
(``csrc/``), driven through the C-ABI declared in ``include/tsat.h``.
"""

__version__ = "0.1.0"
