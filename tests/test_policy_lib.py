"""The library's baseline-policy checkpoint sets (host C++, Hopcroft-Tarjan articulation
points) against the oracle's (brute-force articulation points); CPU only."""
import numpy as np
import pytest

from oracle import Instance, policy_K
from workloads import graphs as G

NAMES = {"all": "all", "sqrt": "chen_sqrt", "greedy": "chen_greedy", "ap_sqrt": "ap_sqrt",
         "ap_greedy": "ap_greedy"}


@pytest.mark.parametrize("name", ["chain", "resnet50", "unet", "vgg16", "random"])
def test_checkpoint_sets_match_oracle(name):
    import paper_1910_02653_b200 as cm
    g = {"chain": lambda: G.training_chain(13), "resnet50": G.resnet50, "unet": G.unet,
         "vgg16": G.vgg16, "random": lambda: G.random_training(25, 0.3, 9)}[name]()
    graph = object.__new__(cm.Graph)            # host-side fields only (no device upload)
    graph.n = g.n
    graph.pred_ptr, graph.pred_idx = (np.ascontiguousarray(a, np.int32) for a in g.pred_csr())
    graph.mem = np.ascontiguousarray(g.mem, np.int64)
    inst = Instance.from_graph(g)
    fwd = int(g.mem[: g.L].sum())
    for pol in NAMES:
        for b in ([0] if "greedy" not in pol else [1, fwd // 16, fwd // 5, fwd // 2, fwd + 1]):
            got = {int(v) + 1 for v in np.nonzero(cm.policy_checkpoints(graph, g.L, pol, b))[0]}
            assert got == policy_K(inst, g.L, NAMES[pol], b), (pol, b)
