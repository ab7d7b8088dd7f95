"""Pins the oracle's Rng restatement against streams produced by the reference's own
rng.hpp (compiled unchanged; tests/golden/rng_golden.json, tests/golden/make_golden.py)."""
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "rng_golden.json")))


@pytest.mark.parametrize("stream", G["streams"], ids=lambda s: str(s["seed"]))
def test_rng_streams_match_reference(O, stream):
    r = O.Rng(stream["seed"])
    assert [str(r.next_u64()) for _ in range(8)] == stream["u64"]
    assert [r.uniform() for _ in range(8)] == stream["uniform"]
    assert [r.normal() for _ in range(8)] == stream["normal"]
    assert [r.chi_square3() for _ in range(4)] == stream["chi_square3"]
    assert [r.uniform_index(1000) for _ in range(8)] == stream["uniform_index_1000"]
    assert [r.uniform_index(7) for _ in range(8)] == stream["uniform_index_7"]
    assert [r.uniform(0.0, 6.283185307179586476925287) for _ in range(4)] == stream["uniform_range"]
    assert str(r.derive(17).next_u64()) == stream["derive_17"]


def test_derive_seed_matches_reference(O):
    for s, t, v in G["derive_seed"]:
        assert str(O.derive_seed(int(s), int(t))) == v


def test_product_rng_matches_reference(W):
    """The product's host-side Rng (used for SGD batches / RFF draws) is the same stream."""
    for stream in G["streams"]:
        r = W.Rng(stream["seed"])
        assert [str(r.next_u64()) for _ in range(8)] == stream["u64"]
        assert [r.uniform() for _ in range(8)] == stream["uniform"]
        assert [r.normal() for _ in range(8)] == stream["normal"]
    for s, t, v in G["derive_seed"]:
        assert str(W.derive_seed(int(s), int(t))) == v
