"""CPU: graph.py semantics equal the reference's (graph.py:114-293) on the
reference's own MLP and transformer graphs -- frontiers of every slice,
partition of every small slice -- when the reference is importable (this
build container; skipped elsewhere)."""

import sys
from pathlib import Path

import pytest

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref():
    if not REF_SRC.is_dir():
        pytest.skip("reference not present")
    sys.path.insert(0, str(REF_SRC))
    try:
        from fpverify import graph as RG, models as RM
    finally:
        sys.path.remove(str(REF_SRC))
    return RG, RM


@pytest.mark.parametrize("model", ["mlp", "transformer"])
def test_frontiers_match_reference(ref, model):
    from paper_2510_16028_b200 import graph as G
    RG, RM = ref
    g = (RM.build_mlp(seed=0) if model == "mlp" else RM.build_transformer(seed=0)).graph
    n = g.n_nodes
    for a in range(n):
        for b in range(a + 1, min(n, a + 40) + 1):
            r, o = RG.frontiers(g, RG.Slice(a, b)), G.frontiers(g, G.Slice(a, b))
            assert (r.in_inputs, r.in_weights, r.in_nodes, r.out_nodes) == \
                (o.in_inputs, o.in_weights, o.in_nodes, o.out_nodes), (a, b)


def test_partition_and_build_graph_match_reference(ref):
    from paper_2510_16028_b200 import graph as G
    RG, RM = ref
    for n in range(2, 9):
        for a in range(6):
            for b in range(a + 1, 40):
                assert [(s.start, s.end) for s in RG.partition(RG.Slice(a, b), n)] == \
                    [(s.start, s.end) for s in G.partition(G.Slice(a, b), n)]
    g = RM.build_transformer(seed=0).graph
    ours = G.build_graph([G.make_node(x.name, x.kind, x.inputs, dict(x.attrs)) for x in g.nodes],
                         list(g.inputs), g.weights, list(g.outputs), allow_extensions=False)
    assert [(x.index, x.name, x.kind, x.inputs, x.attrs) for x in ours.nodes] == \
        [(x.index, x.name, x.kind, tuple(x.inputs), tuple(x.attrs)) for x in g.nodes]
    with pytest.raises(ValueError, match="producers must precede"):
        G.build_graph([G.make_node("a", "neg", ["node:0"])], [], {}, ["node:0"])
