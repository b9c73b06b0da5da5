"""CPU checks of the lockstep parity metric (tests/parity.py)."""
import numpy as np

from tests.parity import parity_error


def _state(seed, zero_comp=None):
    rng = np.random.default_rng(seed)
    s = {(0, 0, 0): rng.uniform(0.5, 2.0, (4, 8, 8)), (1, 1, 0): rng.uniform(0.5, 2.0, (4, 8, 8))}
    if zero_comp is not None:
        for v in s.values():
            v[zero_comp] = 0.0
    return s


def test_identical_states_have_zero_error():
    s = _state(1)
    e, rel = parity_error(s, {k: v.copy() for k, v in s.items()})
    assert e == 0.0 and np.all(rel == 0.0)


def test_per_component_max_norm():
    so = _state(2)
    sg = {k: v.copy() for k, v in so.items()}
    sg[(1, 1, 0)][3, 2, 5] += 1e-12
    mx3 = max(np.abs(v[3]).max() for v in so.values())
    e, rel = parity_error(so, sg)
    assert np.isclose(e, 1e-12 / mx3, rtol=1e-3) and rel[:3].max() == 0.0


def test_identically_zero_component_must_be_exactly_zero():
    so = _state(3, zero_comp=2)
    sg = {k: v.copy() for k, v in so.items()}
    assert parity_error(so, sg)[0] == 0.0
    sg[(0, 0, 0)][2, 4, 4] = 1e-300   # any non-zero value where the oracle's component is identically zero
    assert parity_error(so, sg)[0] == np.inf


def test_rounding_level_component_uses_the_floor():
    so = _state(4)
    for v in so.values():
        v[2] *= 1e-17   # zero up to rounding, not identically zero
    sg = {k: v.copy() for k, v in so.items()}
    sg[(0, 0, 0)][2, 1, 1] += 1e-17
    e, _ = parity_error(so, sg)
    mx = max(np.abs(v).max() for v in so.values())
    assert np.isfinite(e) and e <= 1e-17 / (1e-3 * mx) * (1 + 1e-9)
