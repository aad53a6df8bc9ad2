"""Cost calibration (paper_2504_14519_b200/calibrate.py): fitting the
reference CostModel (workload.cpp:162-187) to a step timeline recovers the
costs exactly when the timeline is the reference simulator's own, and the
calibrated simulate() then reproduces that timeline's bubble."""
import pytest

from paper_2504_14519_b200 import calibrate as CAL
from paper_2504_14519_b200 import plan as P


@pytest.mark.parametrize("p,m,n,cost", [(2, 2, 4, (1.0, 0.25, 2.0, 1.0)), (4, 4, 8, (0.7, 0.05, 2.0, 0.0)),
                                         (8, 4, 8, (1.3, 0.11, 1.5, 0.5))])
def test_fit_recovers_the_reference_costs(p, m, n, cost):
    S = 16 * n
    sim = P.simulate(p, 1, m, n, "off", cost=cost, seq_len=S)
    per_dev = [[tuple(x) for x in dev] for dev in sim["timeline"]]
    fit = CAL.fit_costs(p, 1, m, n, S, per_dev)
    for got, want in zip((fit["alpha"], fit["beta"], fit["bwd_in"], fit["bwd_w"]), cost):
        assert got == pytest.approx(want, rel=1e-9, abs=1e-12)
    out = CAL.predict(p, 1, m, n, S, per_dev, modes=("off", "on"))
    assert out["measured"]["bubble"] == pytest.approx(sim["bubble"], rel=1e-12)
    assert out["simulated"]["off"]["bubble"] == pytest.approx(sim["bubble"], rel=1e-9)
    assert out["simulated"]["on"]["bubble"] <= out["simulated"]["off"]["bubble"] + 1e-12
