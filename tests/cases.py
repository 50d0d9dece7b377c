"""Rebuild the golden stepper cases (tests/golden/steppers.json) for either
the oracle (CPU) or the GPU package, from the same descriptors."""

import numpy as np


def oracle_problem(case):
    import cgl_oracle as O
    p = O.Params(**case["params"])
    if case["op"] == "fd":
        d = len(case["extents"])
        mats = [p.diffusion * O.FD_BUILDERS[case["bc"]](n, L) + (p.alpha2 / d) * np.eye(n)
                for n, L in zip(case["extents"], case["lengths"])]
        blocks = [O.KronOp(mats)]
    else:
        sgn = (1, -1) if case["kind"] == "coupled_cubic_quintic" else (0,)
        blocks = [O.FourierOp(O.symbol(case["extents"], case["intervals"], p, s)) for s in sgn]
    return O.Prob(blocks, case["kind"], p)


def gpu_problem(case):
    from paper_2403_02816_b200 import (BlockOperator, CglParameters, FourierGrid, NonlinearSpec, Problem,
                                       build_fd_operator, build_periodic_operator)
    p = CglParameters(**case["params"])
    spec = NonlinearSpec(case["kind"], p)
    if case["op"] == "fd":
        op = build_fd_operator(p, tuple(case["extents"]), tuple(case["lengths"]), case["bc"])
    else:
        grid = FourierGrid(tuple(case["extents"]), tuple(tuple(x) for x in case["intervals"]))
        if spec.components == 2:
            op = BlockOperator([build_periodic_operator(grid, p, 1), build_periodic_operator(grid, p, -1)])
        else:
            op = build_periodic_operator(grid, p)
    return Problem(op, spec)


def inputs(case, arrays):
    i = case["index"]
    return ([arrays[f"s{i}_ic{c}"] for c in range(case["components"])],
            [arrays[f"s{i}_out{c}"] for c in range(case["components"])])
