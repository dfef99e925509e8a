"""The dataflow tile Cholesky (csrc/chol.cu k_chol_dataflow) under different schedules.

The updates of every tile are applied in a fixed step order whatever CTA runs them and whenever,
so the factor -- and everything downstream of it -- must be bit-identical across scheduling
parameters: the high-queue CTA count, the high-class threshold, and the dispensing order.  A
scheduler bug (a task run before one of its inputs, a lost or doubled update) shows up as a
difference here even when the result would still pass a tolerance test.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from precompute.basis import build_basis  # noqa: E402
from precompute.mesh import make_scene  # noqa: E402


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


@pytest.fixture(scope="module")
def c2():
    s = make_scene(2)
    return s, build_basis(s, workers=1)


def run(msim, s, b, env, steps=2):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ctx = msim.context_from_scene(s, b)   # the schedule is fixed when the basis is uploaded
        its = [ctx.timestep().newton_iters for _ in range(steps)]
        x, v = ctx.get_state()
        info = ctx.coarse_info()
    finally:
        for k, val in old.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val
    return its, x, v, info


@pytest.mark.parametrize("env", [{"MSIM_DF_HI": "1"}, {"MSIM_DF_HI": "3", "MSIM_DF_HIDJ": "6"},
                                 {"MSIM_DF_HIDJ": "1"}])
def test_schedule_independent(msim, c2, env):
    s, b = c2
    its0, x0, v0, info = run(msim, s, b, {})
    assert info["ntiles"] >= 8              # a DAG with real concurrency
    its1, x1, v1, _ = run(msim, s, b, env)
    assert its1 == its0
    assert np.array_equal(x1, x0) and np.array_equal(v1, v0)
