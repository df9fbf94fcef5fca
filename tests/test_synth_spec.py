"""SyntheticSpec / generation_slack_actions (workload.py:296-368): validation
messages and the slack arithmetic, against values recorded from the reference
(tests/golden/synth_stats.json).  Host-only."""
from __future__ import annotations

import pytest

import golden_io


def test_spec_validation_messages_match_reference():
    from paper_2605_11381_b200.synth import SyntheticSpec
    errs = golden_io.synth()["spec_errors"]
    assert len(errs) == 10
    for kw, msg in errs:
        with pytest.raises(ValueError) as e:
            SyntheticSpec.from_dict(kw)
        assert str(e.value) == msg


@pytest.mark.parametrize("lat,hz,exp", [(100_000, 30.0, 3), (33_333, 30.0, 1), (33_334, 30.0, 2),
                                        (0, 30.0, 0), (1, 29.97, 1), (500_000, 15.0, 8)])
def test_generation_slack_actions(lat, hz, exp):
    from paper_2605_11381_b200.synth import generation_slack_actions
    assert generation_slack_actions(lat, hz) == exp
