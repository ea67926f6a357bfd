"""Attention binding: which op a runner process serves, its space, and the param mapping.

The reference binding maps shape dims to tensor recipes and a Triton grid
(ref/pkg/runner/src/ktune_triton_runner/binding.py:40-163); it cannot express cu_seqlens, page
pools or block tables (binding.py:154-163), so an attention binding names the op instead and the
workload is built from the ShapeKey dims (paper_2505_03780_b200/workload.py).  The invariant the
reference enforces is kept: every space parameter must map to a kernel knob
(binding.py:115-125), and unknown mappings are startup errors.

    {"op": "prefill", "space_file": "../spaces/flash_attention.space.json",
     "config_params": {"BLOCK_M": "BLOCK_M", ...}, "seed": 0}
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path

from .. import configspace

# kernel knobs each op understands (attention.PREFILL_PARAMS / DECODE_PARAMS)
KNOBS = {
    "prefill": ("BLOCK_M", "BLOCK_N", "num_warps", "num_stages", "waves_per_eu", "PRE_LOAD_V"),
    "decode": ("num_splits", "num_stages", "TILE_N"),
}


class BindingError(Exception):
    pass


@dataclass(frozen=True)
class AttentionBinding:
    op: str
    space_path: Path
    space: configspace.ConfigSpace
    config_params: dict
    seed: int = 0

    @classmethod
    def load(cls, path) -> "AttentionBinding":
        path = Path(path)
        try:
            doc = json.loads(path.read_text())
        except (OSError, json.JSONDecodeError) as e:
            raise BindingError(f"cannot read binding {path}: {e}") from None
        op = doc.get("op")
        if op not in KNOBS:
            raise BindingError(f"binding 'op' must be one of {sorted(KNOBS)}, got {op!r}")
        if "space_file" not in doc:
            raise BindingError("binding is missing 'space_file'")
        space_path = (path.parent / doc["space_file"]).resolve()
        if not space_path.is_file():
            raise BindingError(f"space file does not exist: {space_path}")
        try:
            space = configspace.parse_space_file(space_path)
        except (configspace.SpaceError, OSError) as e:
            raise BindingError(f"space file {space_path} is malformed: {e}") from None
        cp = dict(doc.get("config_params") or {})
        unmapped = [p for p in space.param_names() if p not in cp]
        if unmapped:
            raise BindingError(f"space parameter {unmapped[0]!r} is not mapped to a kernel hyperparameter")
        unknown = [p for p in cp if p not in space.param_names()]
        if unknown:
            raise BindingError(f"config_params maps {unknown[0]!r}, which is not in the space")
        bad = [k for k in cp.values() if k not in KNOBS[op]]
        if bad:
            raise BindingError(f"{op} kernels have no knob {bad[0]!r} (known: {list(KNOBS[op])})")
        return cls(op, space_path, space, cp, int(doc.get("seed", 0)))

    def kernel_config(self, config: dict) -> dict:
        return {knob: config[param] for param, knob in self.config_params.items()}

    def space_digest(self) -> str:
        """Canonical ktune space digest (whitespace edits do not bust the cache)."""
        return self.space.digest


def kernel_source_digest() -> str:
    """SHA-256 over every kernel/ABI source AND the built library (hashing Python alone would
    miss kernel edits)."""
    pkg = Path(__file__).resolve().parents[1]
    h = hashlib.sha256()
    files = sorted((pkg / "csrc").glob("*.cu*")) + [pkg.parent / "include" / "b200attn.h",
                                                     pkg / "_lib" / "libb200attn.so"]
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes() if f.exists() else b"<missing>")
    return h.hexdigest()
