"""Record the reference ktune's digests/cardinalities so tests/test_configspace.py can pin our
independent implementation against them on machines without /root/reference.

Run HERE:  python tests/golden/make_ktune_digests.py   (imports ref/pkg/src/ktune read-only)
"""
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
from ktune import configspace as R, expr as E  # noqa: E402

ROOT = Path(__file__).resolve().parents[2]
spaces = {
    "ref:flash_attention": REF / "ktune/fixtures/flash_attention.space.json",
    "ref:rms_norm": REF / "ktune/fixtures/rms_norm.space.json",
    "ref:vector_add": REF / "ktune/fixtures/vector_add.space.json",
    "flash_attention": ROOT / "paper_2505_03780_b200/spaces/flash_attention.space.json",
    "paged_decode": ROOT / "paper_2505_03780_b200/spaces/paged_decode.space.json",
}
out = {"spaces": {}, "exprs": {}, "shapes": {}}
for key, path in spaces.items():
    s = R.parse_space_file(path)
    cfgs = list(R.enumerate_configs(s))
    out["spaces"][key] = {
        "doc": json.loads(path.read_text()),
        "digest": s.digest,
        "cardinality": list(R.cardinality(s)),
        "first_configs": [c.assignments for c in cfgs[:5]],
        "config_digests_sha": R.digest_of([c.digest for c in cfgs]),
    }
for t in ["a+b*c-d/e%f", "!(A && B) || C == D", "-a < -(b)", "a<b==c", "BLOCK_M % 32 == 0 || num_warps < 4",
          "((a))+1", "!(PRE_LOAD_V && num_stages > 2)"]:
    out["exprs"][t] = E.canonical(E.parse_expr(t))
for dims in [{"op": "prefill", "batch_size": 1, "seq_len": 512}, {"seq_len": 4096, "batch_size": 64, "dtype": "bfloat16"}]:
    out["shapes"][json.dumps(dims)] = R.ShapeKey.from_dims(dims).digest
(Path(__file__).parent / "ktune_digests.json").write_text(json.dumps(out, indent=1, sort_keys=True))
print("ok")
