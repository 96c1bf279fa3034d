"""Product partitioner vs the reference goldens (fp/partition.py:57-132)."""

import pytest

from golden_util import load
from paper_2509_09560_b200 import plan_stages, split_generation, split_perception
from paper_2509_09560_b200.errors import InvalidStageCount, TooManyStages


def test_generation_goldens():
    for c in load("partition")["generation"]:
        assert split_generation(c["n"], c["stages"], c["alpha"]) == c["counts"], c


def test_perception_goldens():
    for c in load("partition")["perception"]:
        assert [list(r) for r in split_perception(c["costs"], c["stages"])] == c["ranges"], c


def test_fault_hook(monkeypatch):
    f = load("partition")["fault_truncate"]
    monkeypatch.setenv("FRAMEPIPE_ROUNDING_FAULT", "truncate")
    assert split_generation(100, 4, 0.5) == f["counts"] == [10, 16, 28, 46]


def test_errors():
    with pytest.raises(InvalidStageCount):
        split_generation(3, 4, 0.0)
    with pytest.raises(InvalidStageCount):
        split_generation(0, 1, 0.0)
    with pytest.raises(TooManyStages):
        split_perception([1.0, 1.0], 3)


def test_plan_stage_starts():
    plan = plan_stages([1.0, 1.0], 2, 100, 4, 0.5)
    assert plan.generation_stages == (10, 17, 27, 46)
    assert plan.stage_starts() == (0, 10, 27, 54)
    assert plan.to_dict()["generation_stages"] == [10, 17, 27, 46]
