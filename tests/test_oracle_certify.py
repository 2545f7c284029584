"""Pins of the O(E) LP-duality certificate (oracle/certify.py).

`dual_certificate_batch` is the checker run on every GPU frame, so it is pinned here against
  * the scalar `dual_certificate` (written check by check in the order of c.4) on oracle
    decode outputs of config-1 and config-2 frames: same verdict, same min lhs / bound gap;
  * what weak duality fixes: on a correct oracle output UB - LB is tiny and LB <= OPT <= UB
    with OPT the oracle objective (the LP optimum, Thm 2c);
  * wrong answers it must reject: a flipped hard decision (Alg. 2 then finds a violated cut,
    P:119-120), a dual-infeasible y (y_j > 0 breaks z_{n+j} = -y_j >= 0, dual LP P:418-428 read
    as G4), a u outside the box, a y scaled so the bound gap opens, a z = c - A^T y < 0.
"""
import numpy as np
import pytest

from oracle.certify import dual_certificate, dual_certificate_batch
from oracle.lp import malp_decode
from synth import config_code, config_frames


def _oracle_outputs(cfg, snr_idx, frames):
    code = config_code(cfg)
    fb = config_frames(cfg, snr_idx, frames=frames, code=code) if cfg == 2 else \
        config_frames(cfg, frames=frames, code=code)
    outs = [malp_decode(code, fb.llr[f]) for f in range(fb.F)]
    u = np.array([o["u"] for o in outs])
    y = np.array([o["y"] for o in outs])
    masks = np.array([o["masks"] for o in outs], dtype=np.uint16)
    obj = np.array([o["obj"] for o in outs])
    status = np.array([o["status"] for o in outs])
    return code, fb.llr, u, y, masks, obj, status


@pytest.fixture(scope="module")
def c1():
    return _oracle_outputs(1, 0, range(16))


@pytest.fixture(scope="module")
def c2():
    return _oracle_outputs(2, 2, range(4))


def _agree(code, llr, u, y, masks):
    b = dual_certificate_batch(code, llr, u, y, masks)
    for f in range(u.shape[0]):
        s = dual_certificate(code, llr[f], u[f], y[f], masks[f])
        assert bool(b["ok"][f]) == s["ok"], (f, s["reasons"])
        assert b["min_lhs"][f] == pytest.approx(s["min_lhs"], abs=1e-12)
        assert b["gap"][f] == pytest.approx(s["gap"], abs=1e-9 * (1 + abs(s["UB"])))
        assert b["UB"][f] == pytest.approx(s["UB"], rel=1e-13, abs=1e-12)
        assert b["LB"][f] == pytest.approx(s["LB"], rel=1e-12, abs=1e-9)
    return b


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_batch_equals_scalar_and_accepts_oracle_outputs(which, request):
    code, llr, u, y, masks, obj, status = request.getfixturevalue(which)
    b = _agree(code, llr, u, y, masks)
    conv = status == 0
    assert conv.sum() >= 3
    assert np.all(b["ok"][conv])
    # weak duality brackets the LP optimum: LB <= c^T x* <= UB, gamma^T u = c^T x + sum_{gamma<0} gamma
    const = np.where(llr < 0, llr, 0.0).sum(axis=1)
    assert np.all(b["LB"][conv] + const[conv] <= obj[conv] + 1e-9)
    assert np.all(obj[conv] <= b["UB"][conv] + const[conv] + 1e-9)


def test_rejects_flipped_bit(c1):
    code, llr, u, y, masks, obj, status = c1
    f = int(np.nonzero(status == 0)[0][0])
    u2 = u[f:f + 1].copy()
    i = int(np.argmax(np.abs(llr[f])))
    u2[0, i] = 1.0 - np.round(u2[0, i])
    b = _agree(code, llr[f:f + 1], u2, y[f:f + 1], masks[f:f + 1])
    assert not b["ok"][0]
    assert b["min_lhs"][0] < 1.0 - 1e-3 or b["gap"][0] > 1e-3   # cut violated or bound opened


def test_rejects_dual_infeasible_y(c1):
    code, llr, u, y, masks, obj, status = c1
    f = next(f for f in range(len(status)) if status[f] == 0 and (masks[f] >> 15).any())
    j = int(np.nonzero(masks[f] >> 15)[0][0])
    y2 = y[f:f + 1].copy()
    y2[0, j] = 0.5                        # y_j > 0  <=>  slack dual z_{n+j} = -y_j < 0
    b = _agree(code, llr[f:f + 1], u[f:f + 1], y2, masks[f:f + 1])
    assert not b["ok"][0]


def test_rejects_negative_reduced_cost(c1):
    code, llr, u, y, masks, obj, status = c1
    f = next(f for f in range(len(status)) if status[f] == 0 and (masks[f] >> 15).any())
    j = int(np.nonzero(masks[f] >> 15)[0][0])
    y2 = y[f:f + 1].copy()
    y2[0, j] -= 10.0 * (1.0 + np.abs(llr[f]).max())   # y stays <= 0, but |y_j| > c_i makes some z_i < 0
    b = _agree(code, llr[f:f + 1], u[f:f + 1], y2, masks[f:f + 1])
    assert not b["ok"][0]


def test_rejects_box_and_gap(c1):
    code, llr, u, y, masks, obj, status = c1
    f = int(np.nonzero(status == 0)[0][0])
    u2 = u[f:f + 1].copy()
    u2[0, 0] = 1.01 if u2[0, 0] > 0.5 else -0.01
    b = _agree(code, llr[f:f + 1], u2, y[f:f + 1], masks[f:f + 1])
    assert not b["ok"][0]
    # zero duals: dual feasible (z = c >= 0) but LB = 0 while UB = c^T x > 0 -> bound gap
    if np.abs(llr[f]).min() > 0:
        b = _agree(code, llr[f:f + 1], u[f:f + 1], np.zeros_like(y[f:f + 1]), masks[f:f + 1])
        x = np.where(llr[f] < 0, 1 - u[f], u[f])
        if (np.abs(llr[f]) * x).sum() > 1e-3:
            assert not b["ok"][0]
