"""FlopCounter parity: the flops charged at the GEMM / block-solve / GEMV sites of
one exact solve and one Woodbury solve equal the analytic model, as the reference's own
instrumented-vs-analytic test requires (ref:tests/test_subdomain.py:149-159; charge sites
ref:subdomain.py:170-172, 281-282, ref:transform.py:98-100)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand_field(box, seed):
    from paper_2508_07193_b200 import FieldVector
    return FieldVector(box, np.random.default_rng(seed).uniform(-1.0, 1.0, box.dof))


@pytest.mark.parametrize("extents", [(3, 3, 3), (4, 5, 6)])
def test_instrumented_flops_match_analytic_model(extents):
    from paper_2508_07193_b200 import Box, FlopCounter, OperatorParams, exact_solve, precompute, solve
    box = Box(*extents)
    data = precompute(OperatorParams(box, 0.25))
    c = FlopCounter()
    exact_solve(data, rand_field(box, 6), counter=c)
    assert c.total == data.cost.flops_per_exact_solve
    c.reset()
    solve(data, rand_field(box, 7), counter=c)
    assert c.total == data.cost.flops_per_solve
    assert c.gemv == data.cost.flops_per_correction


def test_flop_totals_known_answers():
    """ref:tests/test_subdomain.py:162-182 and SURVEY §0 fact 5 (191,038,248 at 34^3)."""
    from paper_2508_07193_b200 import Box, analytic_cost, correction_size
    c32 = analytic_cost(Box(32, 32, 32), correction_size(Box(32, 32, 32)))
    assert c32.flops_total == 151_584_768
    c34 = analytic_cost(Box(34, 34, 34), correction_size(Box(34, 34, 34)))
    assert c34.flops_per_solve == 191_038_248
