"""This repo's uniform depolarizing transformer against the REAL reference's
output (ref gstab/noise.py:104-194): byte-identical noisy texts for every
BASELINE workload (fixtures written by tests/golden/make_golden_noise.py)."""

import gzip
import json
import os

import pytest

from paper_2512_23037_b200 import parse_circuit
from paper_2512_23037_b200.noise import apply_noise_model

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "noise_texts.json.gz")


def _cases():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_transformer_byte_equal_to_reference(case):
    ours = apply_noise_model(parse_circuit(case["base"]), case["p"]).serialize()
    assert ours == case["noisy"]


def test_fixtures_cover_the_generators():
    """The fixture bases are exactly what the generators emit today."""
    import sys
    sys.path.insert(0, os.path.dirname(GOLDEN))
    from make_golden_noise import workloads
    got = {c["name"]: c["base"] for c in _cases()}
    for name, prog, _p in workloads():
        assert parse_circuit(got[name]).serialize() == prog.serialize(), name
