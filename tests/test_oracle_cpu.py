"""The CPU payload restatement (oracle/kvx_oracle.c) checked on its own, on
CPU: against independent numpy restatements of the same operations and
against committed golden digests of its page contents
(tests/golden/fill_digests.json, made by tests/golden/make_fill_golden.py).

The reference stores no bytes, so there are no reference
golden vectors for page contents; the digests pin the oracle's own content
function across rounds (the GPU kernels must match it bit for bit).
"""
import hashlib
import json

import numpy as np
import pytest

from conftest import ROOT

import oracle.oracle as O

GOLDEN = ROOT / "tests" / "golden" / "fill_digests.json"
LAYOUTS = {"tiny_f32": O.Layout(4, 64, 16, 0), "llama_bf16": O.Layout(8, 128, 16, 1)}


def page_bytes(l):
    return 2 * l.num_kv_heads * l.block_tokens * l.head_dim * (2 if l.dtype == 1 else 4)


def fill(layout, tags, seed, mode):
    pb = page_bytes(layout)
    pool = np.zeros((len(tags), pb), np.uint8)
    O.fill_pages(pool, pb, np.arange(len(tags), dtype=np.uint32), tags, seed, layout, mode)
    return pool


def test_splitmix64_known_answers():
    # splitmix64 reference values (Steele, Lea & Flood; state starts at x)
    assert O.payload().kvxo_splitmix64(0) == 0xE220A8397B1DCDAF
    assert O.payload().kvxo_splitmix64(1) == 0x910A2DEC89025CC1


@pytest.mark.parametrize("name", list(LAYOUTS))
@pytest.mark.parametrize("mode", [0, 1])
def test_fill_matches_golden_digests(name, mode):
    golden = json.loads(GOLDEN.read_text())
    tags = O.tags_array([0, 3, 7, 9], [0, 1, 31, 79], [0, 5, 511, 2047])
    pool = fill(LAYOUTS[name], tags, 20261017, mode)
    assert hashlib.sha256(pool.tobytes()).hexdigest() == golden[f"{name}_mode{mode}"]


def test_fill_values_are_the_stated_distribution():
    pool = fill(LAYOUTS["tiny_f32"], O.tags_array(1, 2, np.arange(64)), 5, 1)
    v = pool.view(np.float32)
    assert np.all(np.abs(v) < 1.7321) and abs(v.mean()) < 0.02 and abs(v.std() - 1.0) < 0.02
    bf = fill(LAYOUTS["llama_bf16"], O.tags_array(1, 2, np.arange(8)), 5, 1).view(np.uint16)
    f = (bf.astype(np.uint32) << 16).view(np.float32)
    assert np.all(np.abs(f) <= 1.7344) and abs(f.std() - 1.0) < 0.02


def test_pack_unpack_copy_are_the_block_table_permutation():
    rng = np.random.default_rng(3)
    pb = 4096
    pool = rng.integers(0, 256, (50, pb), dtype=np.uint8)
    ids = rng.permutation(50)[:20].astype(np.uint32)
    buf = np.zeros(20 * pb, np.uint8)
    O.pack(pool, pb, ids, buf)
    assert np.array_equal(buf.reshape(20, pb), pool[ids])
    dst = np.zeros_like(pool)
    dids = rng.permutation(50)[:20].astype(np.uint32)
    O.unpack(dst, pb, dids, buf)
    assert np.array_equal(dst[dids], pool[ids])
    dst2 = np.zeros_like(pool)
    O.copy_pages(pool, ids, dst2, dids, pb)
    assert np.array_equal(dst2, dst)


def test_append_writes_one_token_slot_per_head():
    l = LAYOUTS["tiny_f32"]
    pb = page_bytes(l)
    pool = np.zeros((4, pb), np.uint8)
    k = np.arange(2 * 4 * 64, dtype=np.float32).reshape(2, 4, 64)
    v = -k
    O.append_kv(pool, l, np.array([3, 1], np.uint32), np.array([5, 15], np.int32), k, v)
    view = pool.view(np.float32).reshape(4, 2, 4, 16, 64)  # [page][K|V][head][tok][d]
    assert np.array_equal(view[3, 0, :, 5], k[0]) and np.array_equal(view[3, 1, :, 5], v[0])
    assert np.array_equal(view[1, 0, :, 15], k[1]) and np.array_equal(view[1, 1, :, 15], v[1])
    assert np.count_nonzero(view[3, :, :, [i for i in range(16) if i != 5]]) == 0


@pytest.mark.parametrize("name", list(LAYOUTS))
def test_attention_oracle_matches_independent_numpy(name):
    """kvxo_decode_attention vs a numpy float64 restatement (gather pages by
    block table, softmax(q.K^T * scale) V per query head, GQA grouping)."""
    l = LAYOUTS[name]
    pb = page_bytes(l)
    rng = np.random.default_rng(11)
    batch, hq, ctx = 3, 2 * l.num_kv_heads, np.array([40, 1, 33], np.int32)
    max_blocks = 3
    pages = batch * max_blocks
    pool = fill(l, O.tags_array(0, 0, np.arange(pages)), 9, 1)
    tables = rng.permutation(pages).astype(np.uint32).reshape(batch, max_blocks)
    if l.dtype == 1:
        qf = rng.standard_normal((batch, hq, l.head_dim)).astype(np.float32)
        q = ((qf.view(np.uint32) + 0x7FFF + ((qf.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
        q64 = (q.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        kv = (pool.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    else:
        q = rng.standard_normal((batch, hq, l.head_dim)).astype(np.float32)
        q64 = q.astype(np.float64)
        kv = pool.view(np.float32).astype(np.float64)
    kv = kv.reshape(pages, 2, l.num_kv_heads, l.block_tokens, l.head_dim)
    scale = float(np.float32(1.0) / np.sqrt(np.float32(l.head_dim)))
    got = O.decode_attention(pool, l, hq, tables, ctx, q, scale)
    g = hq // l.num_kv_heads
    for b in range(batch):
        toks = np.arange(ctx[b])
        pg, slot = tables[b][toks // l.block_tokens], toks % l.block_tokens
        for h in range(hq):
            K = kv[pg, 0, h // g, slot]
            V = kv[pg, 1, h // g, slot]
            s = K @ q64[b, h] * scale
            p = np.exp(s - s.max())
            ref = (p / p.sum()) @ V
            assert np.allclose(got[b, h], ref, rtol=1e-12, atol=1e-12)
