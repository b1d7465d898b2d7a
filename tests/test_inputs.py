"""The seeded synthetic inputs (synth/nrr_synth.hpp) built
through the oracle alone equal, bit for bit, the ones the product's setup
builds: the bench's reference arm generates its inputs without loading
libnrr_b200.so and still times the same workload."""
import dataclasses

import numpy as np
import pytest

from oracle import binding as O
from paper_2206_03410_b200 import registration as R


@pytest.mark.parametrize("config,kw", [(0, dict(scale=0.2)), (1, dict(scale=0.05)), (2, dict(scale=0.1)),
                                       (3, dict(seed=4007, scale=0.25)), (4, dict(scale=0.01))])
def test_oracle_inputs_equal_product_inputs(config, kw):
    a = O.make_problem(config, **kw)
    b = R.make_problem(config, **kw)
    assert np.array_equal(a.source, b.source)
    assert np.array_equal(a.target, b.target)
    assert a.src_avg_edge_length == b.src_avg_edge_length
    for f in dataclasses.fields(b.graph):
        assert np.array_equal(np.asarray(getattr(a.graph, f.name)), np.asarray(getattr(b.graph, f.name))), f.name


def test_graph_multipliers_agree():
    assert O.GRAPH_MULT == R.GRAPH_MULT


def test_synth_rejects_bad_arguments():
    with pytest.raises(O.OracleError):
        O.synth(7)
    with pytest.raises(R.capi.ConfigError):
        R.synth(2, scale=0.0)
