"""Snapshot text format (snapshot.hpp / snapshot.cpp): the C restatement and the product's parser
against fixtures from the reference itself (tests/golden/snapshots.json, make_golden.py)."""
import json
import os

import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "snapshots.json")))


@pytest.mark.parametrize("case", GOLD["serialize"], ids=lambda c: f"{c['h']}x{c['w']}")
def test_port_serialize_matches_reference(case):
    fire = np.array(case["fire"], np.uint8).reshape(case["h"], case["w"])
    agent = tuple(case["agent"]) if case["agent"] else None
    assert O.snapshot_text(O.port(), "port", fire, case["step"], agent).decode() == case["text"]


@pytest.mark.parametrize("case", GOLD["parse"], ids=lambda c: str(len(c["text"])))
def test_parse_matches_reference(case):
    """ebl_snapshot_parse (host code of the product library; no device needed)."""
    if case["ok"]:
        layer, step, agent = eb.parse_snapshot(case["text"])
        assert layer.shape == (case["h"], case["w"]) and step == case["step"]
        assert layer.ravel().tolist() == case["layer"]
        assert agent == (tuple(case["agent"]) if case["agent"] else None)
    else:
        with pytest.raises(eb.FileError) as ei:
            eb.parse_snapshot(case["text"])
        assert str(ei.value).endswith(case["error"])


def test_round_trip_serialize_parse():
    rs = np.random.default_rng(5)
    fire = rs.integers(0, 3, (9, 31)).astype(np.uint8)
    text = O.snapshot_text(O.port(), "port", fire, 123, (4, 30, 2))
    layer, step, agent = eb.parse_snapshot(text)
    assert np.array_equal(layer, fire) and step == 123 and agent == (4, 30, 2)
