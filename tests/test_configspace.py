"""Our ktune-compatible config space vs the reference's recorded digests
(tests/golden/ktune_digests.json, made by tests/golden/make_ktune_digests.py)."""
import json
from pathlib import Path

import pytest

from paper_2505_03780_b200 import configspace as M

G = json.loads((Path(__file__).parent / "golden" / "ktune_digests.json").read_text())


@pytest.mark.parametrize("key", sorted(G["spaces"]))
def test_space_digest_cardinality_enumeration(key):
    rec = G["spaces"][key]
    s = M.parse_space(json.dumps(rec["doc"]))
    assert s.digest == rec["digest"]
    assert list(M.cardinality(s)) == rec["cardinality"]
    cfgs = list(M.enumerate_configs(s))
    assert [c.assignments for c in cfgs[:5]] == rec["first_configs"]
    assert M.digest_of([c.digest for c in cfgs]) == rec["config_digests_sha"]


def test_flash_attention_space_616():
    s = M.parse_space_file(Path(M.__file__).parent / "spaces" / "flash_attention.space.json")
    assert M.cardinality(s) == (1600, 616)  # ref/pkg/tests/test_fixtures.py:20-26


@pytest.mark.parametrize("text", sorted(G["exprs"]))
def test_canonical_constraint_text(text):
    assert M.canonical_text(M.parse_expr(text)) == G["exprs"][text]


def test_shape_digests():
    for dims, dg in G["shapes"].items():
        assert M.ShapeKey.from_dims(json.loads(dims)).digest == dg


def test_whitespace_invariant_digest():
    a = '{"name":"s","params":[{"name":"A","kind":"int-list","values":[1,2,3]}],"constraints":["A<3"]}'
    b = '{ "name": "s", "params": [ {"kind": "int-list", "name": "A", "values": [1, 2, 3]} ],\n "constraints": ["((A) < 3)"] }'
    assert M.parse_space(a).digest == M.parse_space(b).digest


def test_c_semantics_and_errors():
    env = {"a": -7, "b": 2, "t": True}
    ev = lambda t: M.compile_expr(M.parse_expr(t))(env)  # noqa: E731
    assert ev("a / b") == -3 and ev("a % b") == -1 and ev("0 - a % b") == 1
    assert ev("t || (a / 0 == 1)") is True  # short circuit
    with pytest.raises(M.ConstraintEvalError):
        ev("a / (b - 2)")
    with pytest.raises(M.SpaceError):
        M.parse_space('{"name":"s","params":[{"name":"A","kind":"boolean"}],"constraints":["A + 1 > 0"]}')
    with pytest.raises(M.SpaceError):
        M.parse_space('{"name":"s","params":[{"name":"A","kind":"boolean"}],"constraints":["B"]}')
    with pytest.raises(M.SpaceError):
        M.parse_space('{"name":"s","params":[{"name":"A","kind":"pow2-range","lo":3,"hi":8}]}')


def test_validate_config():
    s = M.parse_space_file(Path(M.__file__).parent / "spaces" / "flash_attention.space.json")
    ok, bad = M.validate_config(s, {"BLOCK_M": 128, "BLOCK_N": 256, "num_warps": 4, "num_stages": 2,
                                     "waves_per_eu": 1, "PRE_LOAD_V": True})
    assert not ok and "BLOCK_M >= BLOCK_N" in bad
    with pytest.raises(M.SpaceError):
        M.validate_config(s, {"BLOCK_M": 128})
