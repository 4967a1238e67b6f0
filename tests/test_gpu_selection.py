"""Remask-selection parity at BASELINE.json configs[0-2] against the fp64 CPU
oracle over EVERY masked row (north_star: "remask selections bit-exact").
Every case asserts ZERO mismatches: the device's committed set equals the
fp64 rule's (highest confidence, ties -> lower position). fp32 accumulation
cannot order rows whose fp64 confidences differ by less than its own error
(measured up to 3.4e-5 relative at d 4096), so the record also counts the rows
inside bands of 1e-6 and of twice the measured error around the k-th
confidence (scripts/selection_parity.py writes them to profiles/). Reference: the count schedule
mosaic/workload.py:140-146 and the `commit` op :315 (memory-only there; rule
restated in SURVEY.md §8a a10)."""
import pytest
import torch

import selection_cases as sc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(native_lib):
    return torch.device("cuda", 0)


def test_selection_parity_tiny_config(dev):
    """configs[0]: not vacuous -- with rotary positions the masked rows differ,
    and fewer than 5% of them fall inside the band."""
    rec = sc.tiny_case(dev)
    sc.check(rec)
    assert rec["executor_commit_equals_head"]
    assert rec["band_rows"] < 0.05 * rec["M"], rec


@pytest.mark.parametrize("name,layout", [("llada_32k", "scattered"), ("dream_128k", "suffix")])
def test_selection_parity_full_size(dev, name, layout):
    """configs[1] / configs[2]: every one of the 16384 / 65536 masked rows
    against fp64 (the other layout of each runs in scripts/selection_parity.py)."""
    rec = sc.head_case(dev, name, layout)
    sc.check(rec)
