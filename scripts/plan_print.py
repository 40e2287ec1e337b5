"""Print the planner's choice (vlut_plan_ws) for shapes (development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401
import paper_2512_06443_b200 as v  # noqa: E402
if len(sys.argv) > 1:
    v.lib_path = sys.argv[1]
for (M, K, N, g) in [(6912, 2560, 256, 4), (6912, 2560, 128, 4), (6912, 2560, 2048, 4), (2560, 6912, 2048, 4),
                     (2560, 2560, 2048, 4), (4096, 4096, 1024, 4), (4096, 14336, 1024, 4), (3840, 2560, 2048, 4),
                     (3072, 23040, 1024, 5), (3072, 23040, 256, 5), (14336, 4096, 1024, 4)]:
    print((M, K, N, g), v.plan_ws(M, K, N, g))
