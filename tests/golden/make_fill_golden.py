"""Regenerates tests/golden/fill_digests.json: sha256 of the oracle's page
contents (oracle/kvx_oracle.c kvxo_fill_pages) for fixed tags and seed, both
fill modes, both page layouts. Run: python tests/golden/make_fill_golden.py"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle.oracle as O  # noqa: E402

LAYOUTS = {"tiny_f32": O.Layout(4, 64, 16, 0), "llama_bf16": O.Layout(8, 128, 16, 1)}
out = {}
for name, l in LAYOUTS.items():
    pb = 2 * l.num_kv_heads * l.block_tokens * l.head_dim * (2 if l.dtype == 1 else 4)
    tags = O.tags_array([0, 3, 7, 9], [0, 1, 31, 79], [0, 5, 511, 2047])
    for mode in (0, 1):
        pool = np.zeros((4, pb), np.uint8)
        O.fill_pages(pool, pb, np.arange(4, dtype=np.uint32), tags, 20261017, l, mode)
        out[f"{name}_mode{mode}"] = hashlib.sha256(pool.tobytes()).hexdigest()
(ROOT / "tests" / "golden" / "fill_digests.json").write_text(json.dumps(out, indent=1) + "\n")
print(out)
