"""Paper Fig. 3 on the GPU path (proj/src/bench.cpp:118-235): the three host
exclusion regimes over conventional p2p, 2 ranks x T threads, every message
delivered (counted and the credit round trips completed)."""
import pytest

from paper_2208_13707_b200 import workloads


@pytest.mark.gpu
@pytest.mark.parametrize("regime", [0, 1, 2])
@pytest.mark.parametrize("T", [1, 3])
def test_fig3_regimes_deliver_every_message(regime, T):
    out = workloads.fig3(T, W=8, batches=6, nbytes=8, regime=regime)
    assert out["messages"] == T * 8 * 6
    assert out["msgs_per_s"] > 0
    assert out["regime"] == workloads.REGIMES[regime]


@pytest.mark.gpu
def test_fig3_serial_regime_with_owner_trap(monkeypatch):
    # the serial regime's owner trap armed: one thread per comm never trips it
    monkeypatch.setenv("MPIX_SERIAL_CHECK", "1")
    out = workloads.fig3(2, W=4, batches=4, nbytes=16, regime=2)
    assert out["messages"] == 2 * 4 * 4
