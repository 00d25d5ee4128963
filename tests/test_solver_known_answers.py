"""Device known answers of the MGRIT solver (the reference's
tests/test_mgrit.cpp:252-317): from a broadcast initial guess with tolerance
0, the two-level iterate (i) gets closer to the serial sweep with every
V-cycle and (ii) is at the serial solution (here: the fp32 floor against the
device serial sweep) no later than the cycle bound (N/c_f + 1)/2 + 1 that
F-C-F relaxation's exactness front guarantees -- finite termination, whatever
the layer map. The reference pins the exact cycle counts (16 at c_f = 2, 8 at
c_f = 4) on a scalar system whose coarse grid only converges through that
front; a transformer stack with a small step converges geometrically well
before the front arrives, so the count is an upper bound here."""
import numpy as np
import pytest

from paper_2601_09026_b200 import (LayerParallelEngine, LayerStack, SolveConfig, StackConfig,
                                   State, serial_forward)

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(float(np.abs(b).max()), 1e-300))


@pytest.mark.parametrize("cf", [2, 4])
def test_broadcast_start_reaches_serial_within_cycle_bound(cf):
    L, B, s, d = 64, 2, 8, 32
    st = LayerStack(StackConfig(kind="encoder", d=d, heads=2, ffn=64, n_enc=L), 5)
    z0 = State.from_flat(np.random.default_rng(3).standard_normal(B * s * d), B, s, 0, d)
    serial = np.stack([t.flat() for t in serial_forward(st, z0)])
    bound = (L // cf + 1) // 2 + 1
    errs = []
    for k in range(1, bound + 1):
        eng = LayerParallelEngine(st, SolveConfig(coarsen=cf, levels=2, fwd_iters=k, fwd_tol=0.0,
                                                  warm_start=False))
        errs.append(rel(np.stack([t.flat() for t in eng.forward(z0).traj]), serial))
    floor = 1e-5
    assert errs[-1] < floor, errs  # finite termination within the bound
    for a, b in zip(errs, errs[1:]):  # monotone until the fp32 floor
        assert b < a or b < floor, errs
    assert errs[0] > 100 * floor, errs  # one cycle is not enough: the test has teeth
