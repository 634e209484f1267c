"""CM_TRACE chunk timeline of one 125k-S* call (K1 begin/end, K2 begin/end per chunk, ms)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ["CM_TRACE"] = "1"
import paper_1910_02653_b200 as cm
from workloads import graphs as G, budgets as B
from workloads.device_gen import DeviceGenerator
g = G.resnet50(); graph = cm.Graph.from_workload(g)
N = int(os.environ.get("N", "125000"))
dg = DeviceGenerator(g, "g1", 5, layout="dense")
x = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda"); dg.fill(x, 0)
th = torch.tensor([0.5], device="cuda"); bu = torch.tensor(B.geometric_grid(g, 16), device="cuda")
for mode in ("full",):
    for it in range(3):
        cm.round_and_evaluate(graph, x, th, bu); torch.cuda.synchronize()
    tr = cm.debug_trace()
    print(mode)
    for c, t in enumerate(tr): print(c, ["%.3f" % v for v in t])
