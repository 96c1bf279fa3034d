"""Trace aggregation and comparison artefacts (fp/metrics.py) vs the reference.

`summarize` over every recorded trace (pipelined, sequential, PAR, DEC) must
give the reference's RolloutMetrics field for field (the two device-clock
extras aside), and `compare` must serialise byte-identical JSON / CSV / text
tables.  The golden values were produced by the unmodified reference
(oracle/make_golden.py)."""

import json

import pytest

from golden_util import baseline_cases, load, schedule_cases
from paper_2509_09560_b200 import BaselineMissing, FramepipeError, RolloutMetrics, compare, summarize
from paper_2509_09560_b200.metrics import read_metrics, write_trace_jsonl

CASES = schedule_cases() + baseline_cases()
EXTRA = ("jct_p99", "steady_throughput")


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_summarize_matches_reference(case):
    got = json.loads(summarize(case["trace"]).to_json())
    for k in EXTRA:
        got.pop(k)
    assert got == case["metrics"]


def test_compare_tables_byte_identical():
    by = {c["name"]: c for c in CASES}
    for tab in load("baselines")["compare_tables"]:
        runs = [summarize(by[n]["trace"]) for n in tab["names"]]
        t = compare(runs, names=tab["names"], baseline=tab["baseline"])
        assert t.to_json() == tab["json"]
        assert t.to_csv() == tab["csv"]
        assert t.to_text() == tab["text"]


def test_compare_guards(tmp_path):
    m = summarize(CASES[0]["trace"])
    with pytest.raises(BaselineMissing):
        compare([])
    with pytest.raises(BaselineMissing):
        compare([m], baseline=3)
    other = RolloutMetrics.from_dict(dict(m.to_dict(), engine="b200"))
    with pytest.raises(FramepipeError):
        compare([m, other])
    p = tmp_path / "m.json"
    p.write_text(m.to_json())
    assert read_metrics(p) == m
    write_trace_jsonl(CASES[0]["trace"], tmp_path / "t.jsonl")
    lines = (tmp_path / "t.jsonl").read_text().splitlines()
    assert [json.loads(x) for x in lines] == CASES[0]["trace"]
