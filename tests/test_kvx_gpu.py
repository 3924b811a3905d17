"""Payload parity on the B200: every kvx kernel vs the CPU restatement
(oracle/kvx_oracle.c), through the C ABI (include/kvx.h).

Bar: bit-exact for fill / pack / unpack / page copy / append (byte
permutations); attention within the stated tolerance against an fp64
restatement (parity unpinned by the reference, which only models the step):
  fp32 pages (tiny):    max|err| <= 1e-5 * max(1, |ref|)
  bf16 pages, fp32 out: max|err| <= 2e-3 + 1e-2 * |ref|   (P is rounded to bf16
                        before the PV product, as on any bf16 tensor-core path)
"""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2412_16434_b200 import kvx  # noqa: E402

import oracle.oracle as O  # noqa: E402  (test infrastructure)

TINY = kvx.PageLayout(4, 64, 16, kvx.F32)      # config 1: 2 layers, 4 kv heads, d 64, fp32
LLAMA8B = kvx.PageLayout(8, 128, 16, kvx.BF16)  # configs 2/3: 8 kv heads, d 128, bf16


def olayout(l):
    return O.Layout(l.num_kv_heads, l.head_dim, l.block_tokens, l.dtype)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    return torch.device("cuda:0")


def to_dev(a: np.ndarray, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def filled_pool(layout, num_pages, ids, tags, seed, mode, dev):
    pb = layout.page_bytes()
    pool = kvx.Pool(num_pages, pb, device=0)
    kvx.fill_pages(pool, to_dev(ids.astype(np.int32), dev), to_dev(tags.view(np.int32), dev), len(ids), seed,
                   layout, mode)
    ref = np.zeros((num_pages, pb), np.uint8)
    O.fill_pages(ref, pb, ids, tags, seed, olayout(layout), mode)
    return pool, ref


@pytest.mark.parametrize("layout", [TINY, LLAMA8B], ids=["tiny-f32", "8b-bf16"])
@pytest.mark.parametrize("mode", [kvx.FILL_BITS, kvx.FILL_VALUES])
def test_fill_pages_bit_exact(dev, layout, mode):
    rng = np.random.default_rng(1)
    n = 37
    ids = rng.permutation(64)[:n].astype(np.uint32)
    tags = O.tags_array(rng.integers(0, 9, n), rng.integers(0, 80, n), rng.integers(0, 2048, n))
    pool, ref = filled_pool(layout, 64, ids, tags, 0xC0FFEE, mode, dev)
    torch.cuda.synchronize()
    got = pool.as_tensor().cpu().numpy()
    assert np.array_equal(got[ids], ref[ids])
    if mode == kvx.FILL_VALUES:
        vals = got[ids].view(np.float32 if layout.dtype == kvx.F32 else np.uint16)
        if layout.dtype == kvx.BF16:
            vals = (vals.astype(np.uint32) << 16).view(np.float32)
        assert np.all(np.abs(vals) <= 1.7344) and 0.8 < vals.std() < 1.2


@pytest.mark.parametrize("mode", [kvx.COPY_SM, kvx.COPY_TMA])
@pytest.mark.parametrize("layout,n", [(TINY, 1), (TINY, 24), (LLAMA8B, 0), (LLAMA8B, 1), (LLAMA8B, 333)])
def test_pack_unpack_bit_exact(dev, layout, n, mode):
    pb = layout.page_bytes()
    rng = np.random.default_rng(n)
    pages = 2 * max(n, 1) + 3
    ids = rng.permutation(pages)[:n].astype(np.uint32)
    dst_ids = rng.permutation(pages)[:n].astype(np.uint32)
    tags = O.tags_array(7, rng.integers(0, 32, n), np.arange(n))
    src, ref = filled_pool(layout, pages, ids, tags, 42, kvx.FILL_BITS, dev)
    buf = torch.zeros(max(n, 1) * pb, dtype=torch.uint8, device=dev)
    kvx.pack(src, to_dev(ids.view(np.int32), dev), n, buf, mode)
    ref_buf = np.zeros(max(n, 1) * pb, np.uint8)
    O.pack(ref, pb, ids, ref_buf)
    dst = kvx.Pool(pages, pb, device=0)
    dst.as_tensor().zero_()
    kvx.unpack(dst, to_dev(dst_ids.view(np.int32), dev), n, buf, mode)
    ref_dst = np.zeros((pages, pb), np.uint8)
    O.unpack(ref_dst, pb, dst_ids, ref_buf)
    torch.cuda.synchronize()
    assert np.array_equal(buf.cpu().numpy(), ref_buf)
    assert np.array_equal(dst.as_tensor().cpu().numpy(), ref_dst)


@pytest.mark.parametrize("mode", [kvx.COPY_SM, kvx.COPY_TMA, kvx.COPY_CE])
def test_copy_pages_between_pools_bit_exact(dev, mode):
    layout = LLAMA8B
    pb = layout.page_bytes()
    rng = np.random.default_rng(5)
    n, pages = 200, 260
    def ids_with_run(start):  # unique ids with one consecutive run the copy engines coalesce
        rest = rng.permutation(np.setdiff1d(np.arange(pages), np.arange(start, start + 10)))[:n - 10]
        return np.concatenate([rest[:10], np.arange(start, start + 10), rest[10:]]).astype(np.uint32)
    src_ids, dst_ids = ids_with_run(30), ids_with_run(100)
    tags = O.tags_array(3, 5, np.arange(n))
    src, ref = filled_pool(layout, pages, src_ids, tags, 9, kvx.FILL_VALUES, dev)
    dst = kvx.Pool(pages, pb, device=0)
    dst.as_tensor().zero_()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        if mode == kvx.COPY_CE:
            kvx.copy_pages(src, src_ids, dst, dst_ids, n, mode, stream=s)
        else:
            kvx.copy_pages(src, to_dev(src_ids.view(np.int32), dev), dst, to_dev(dst_ids.view(np.int32), dev), n,
                           mode, stream=s)
    s.synchronize()
    ref_dst = np.zeros((pages, pb), np.uint8)
    O.copy_pages(ref, src_ids, ref_dst, dst_ids, pb)
    assert np.array_equal(dst.as_tensor().cpu().numpy(), ref_dst)


@pytest.mark.parametrize("mode", [kvx.COPY_AUTO, kvx.COPY_SM, kvx.COPY_TMA])
def test_copy_pages_listed_bit_exact(dev, mode):
    """kvx_copy_pages_listed (the payload's per-layer HBM moves): host id
    lists in the launch parameters, 5,000 scattered pages = two launches of
    <= 3,840, every mover; out-of-range ids rejected before any launch."""
    layout = LLAMA8B
    pb = layout.page_bytes()
    rng = np.random.default_rng(23 + mode)
    n, pages = 5000, 5300
    src_ids = rng.permutation(pages)[:n].astype(np.uint32)
    dst_ids = rng.permutation(pages)[:n].astype(np.uint32)
    tags = O.tags_array(6, 1, np.arange(n))
    src, ref = filled_pool(layout, pages, src_ids, tags, 31, kvx.FILL_VALUES, dev)
    dst = kvx.Pool(pages, pb, device=0)
    dst.as_tensor().zero_()
    torch.cuda.synchronize()
    lib = kvx.lib()
    V, U64 = ctypes.c_void_p, ctypes.c_uint64
    lib.kvx_copy_pages_listed.argtypes = [V, V, V, V, U64, ctypes.c_int, ctypes.c_uint32, V]
    s = torch.cuda.Stream()
    rc = lib.kvx_copy_pages_listed(src.handle, src_ids.ctypes.data, dst.handle, dst_ids.ctypes.data, n, mode, 0,
                                   ctypes.c_void_p(s.cuda_stream))
    assert rc == 0, lib.kvx_last_error()
    s.synchronize()
    ref_dst = np.zeros((pages, pb), np.uint8)
    O.copy_pages(ref, src_ids, ref_dst, dst_ids, pb)
    assert np.array_equal(dst.as_tensor().cpu().numpy(), ref_dst)
    bad = dst_ids.copy()
    bad[-1] = pages  # out of range
    assert lib.kvx_copy_pages_listed(src.handle, src_ids.ctypes.data, dst.handle, bad.ctypes.data, n, mode, 0,
                                     ctypes.c_void_p(s.cuda_stream)) == 2


@pytest.mark.parametrize("pattern", ["fragmented", "runs"])
def test_copy_engine_lane_host_pools_bit_exact(dev, pattern):
    """KVX_COPY_CE with host id lists between HBM and a pinned mapped HOST pool
    (the payload's PCIe lanes), both directions: fragmented ids take the
    listed-id SM mover (ids in the launch parameters; 5,000 pages = two
    launches of <= 3,840), long runs one cudaMemcpyAsync per run."""
    layout = LLAMA8B
    pb = layout.page_bytes()
    rng = np.random.default_rng(17)
    n, pages = 5000, 5200
    if pattern == "fragmented":
        src_ids = rng.permutation(pages)[:n].astype(np.uint32)
        host_ids = rng.permutation(pages)[:n].astype(np.uint32)
    else:
        src_ids = np.arange(100, 100 + n, dtype=np.uint32)
        host_ids = np.arange(7, 7 + n, dtype=np.uint32)
    tags = O.tags_array(4, 2, np.arange(n))
    src, ref = filled_pool(layout, pages, src_ids, tags, 21, kvx.FILL_VALUES, dev)
    host = kvx.Pool(pages, pb, host=True)
    back = kvx.Pool(pages, pb, device=0)
    back.as_tensor().zero_()
    torch.cuda.synchronize()  # the fill ran on the legacy stream
    s = torch.cuda.Stream()
    kvx.copy_pages(src, src_ids, host, host_ids, n, kvx.COPY_CE, stream=s)   # D2H
    kvx.copy_pages(host, host_ids, back, src_ids, n, kvx.COPY_CE, stream=s)  # H2D
    s.synchronize()
    got = back.as_tensor().cpu().numpy()
    assert np.array_equal(got[src_ids], ref[src_ids])


@pytest.mark.parametrize("mode", [kvx.COPY_SM, kvx.COPY_TMA])
@pytest.mark.parametrize("cap", [1, 3, 17])
def test_capped_copy_bit_exact(dev, mode, cap):
    """Background migration with the mover's grid capped (kvx_copy_pages_capped):
    fewer CTAs than work items, every page still lands bit-exact."""
    layout = LLAMA8B
    pb = layout.page_bytes()
    rng = np.random.default_rng(cap)
    n, pages = 150, 400
    src_ids = rng.permutation(pages)[:n].astype(np.uint32)
    dst_ids = rng.permutation(pages)[:n].astype(np.uint32)
    src, ref = filled_pool(layout, pages, src_ids, O.tags_array(4, 2, np.arange(n)), 13, kvx.FILL_BITS, dev)
    dst = kvx.Pool(pages, pb, device=0)
    dst.as_tensor().zero_()
    kvx.copy_pages(src, to_dev(src_ids.view(np.int32), dev), dst, to_dev(dst_ids.view(np.int32), dev), n, mode,
                   max_ctas=cap)
    torch.cuda.synchronize()
    ref_dst = np.zeros((pages, pb), np.uint8)
    O.copy_pages(ref, src_ids, ref_dst, dst_ids, pb)
    assert np.array_equal(dst.as_tensor().cpu().numpy(), ref_dst)


@pytest.mark.parametrize("layout", [TINY, LLAMA8B], ids=["tiny-f32", "8b-bf16"])
def test_file_pool_roundtrip_bit_exact(dev, layout, tmp_path):
    """DISK tier as a file: HOST pool -> file -> second HOST pool, in stream
    order on one stream (pwrite then pread as host callbacks), runs of
    consecutive ids coalesced; every page bit-exact, and the file holds the
    pages at page_id * page_bytes. Device pools cannot exchange with a file."""
    pb = layout.page_bytes()
    rng = np.random.default_rng(21)
    n, pages = 50, 64
    host = kvx.Pool(pages, pb, host=True)
    host_np = host.as_tensor().numpy()
    host_np[:] = rng.integers(0, 256, host_np.shape, dtype=np.uint8)
    disk = kvx.Pool.file(tmp_path / "disk.pages", pages, pb)
    src_ids = np.concatenate([np.arange(10, 20), rng.permutation(np.arange(20, pages))[:n - 10]]).astype(np.uint32)
    dst_ids = np.concatenate([np.arange(30, 40), rng.permutation(np.setdiff1d(np.arange(pages), np.arange(30, 40)))[:n - 10]]).astype(np.uint32)
    back = kvx.Pool(pages, pb, host=True)
    back.as_tensor().zero_()
    s = torch.cuda.Stream()
    kvx.copy_pages(host, src_ids, disk, dst_ids, n, kvx.COPY_CE, stream=s)
    kvx.copy_pages(disk, dst_ids, back, src_ids, n, kvx.COPY_CE, stream=s)
    s.synchronize()
    got = back.as_tensor().numpy()
    assert np.array_equal(got[src_ids], host_np[src_ids])
    for i in (0, 17, n - 1):
        assert np.array_equal(disk.read_page(int(dst_ids[i])), host_np[src_ids[i]])
    raw = np.fromfile(tmp_path / "disk.pages", np.uint8).reshape(pages, pb)
    assert np.array_equal(raw[dst_ids], host_np[src_ids])
    dev_pool = kvx.Pool(pages, pb, device=0)
    with pytest.raises(kvx.KvxError):
        kvx.copy_pages(dev_pool, src_ids, disk, dst_ids, n, kvx.COPY_CE)


def test_device_signal_orders_streams(dev):
    """kvx_signal_write / kvx_signal_wait: a consumer stream that waits on a
    flag sees everything the producer stream wrote before setting it (here a
    50 ms spin delays the producer, so without the wait the copy would read
    the old bytes)."""
    flag = torch.zeros(4, dtype=torch.int32, device=dev)
    src = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    dst = torch.empty_like(src)
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(prod):
        torch.cuda._sleep(100_000_000)
        src.fill_(7)
    kvx.signal_write(flag.data_ptr() + 4, 3, prod)
    kvx.signal_wait(flag.data_ptr() + 4, 3, cons)
    with torch.cuda.stream(cons):
        dst.copy_(src)
    torch.cuda.synchronize()
    assert int(flag[1]) == 3 and bool((dst == 7).all())
    with pytest.raises(kvx.KvxError):
        kvx.signal_write(flag.data_ptr() + 2, 1, prod)  # misaligned flag


@pytest.mark.parametrize("batch,ctx", [(1, 8192), (3, 1000), (16, 4096)])
def test_early_prefetch_is_bit_identical(dev, batch, ctx):
    """KVX_ATTN_EARLY_PREFETCH (table + first pages fetched before the PDL
    wait) changes timing only: back-to-back launches — plain and fused-append
    steps — give the same outputs and pool bytes as without it."""
    layout = LLAMA8B
    pb = layout.page_bytes()
    mb = (ctx + 15) // 16
    pages = batch * mb + 4
    rng = np.random.default_rng(batch)
    tables = to_dev(rng.permutation(pages)[:batch * mb].astype(np.int32).reshape(batch, mb), dev)
    lens = to_dev(np.full(batch, ctx, np.int32) - rng.integers(0, 16, batch).astype(np.int32), dev)
    ids = torch.arange(pages, dtype=torch.int32, device=dev)
    tags = torch.stack([ids * 0 + 2, ids * 0, ids], -1).contiguous()
    q = torch.randn(batch, 32, 128, device=dev).to(torch.bfloat16)
    nk = torch.randn(batch, 8, 128, device=dev).to(torch.bfloat16)
    results = []
    for flags in (0, kvx.ATTN_EARLY_PREFETCH):
        pool = kvx.Pool(pages, pb, device=0)
        kvx.fill_pages(pool, ids, tags, pages, 3, layout, kvx.FILL_VALUES)
        att = kvx.Attention(layout, 32, mb, flags=flags)
        ws = torch.zeros(max(att.workspace_bytes(batch, ctx), 1), dtype=torch.uint8, device=dev)
        outs = [torch.empty(batch, 32, 128, dtype=torch.float32, device=dev) for _ in range(4)]
        for i, o in enumerate(outs):  # back to back on one stream: PDL overlaps consecutive launches
            if i % 2:
                att(pool, tables, lens, q, o, batch, ctx, ws, new_k=nk, new_v=nk)
            else:
                att(pool, tables, lens, q, o, batch, ctx, ws)
        torch.cuda.synchronize()
        results.append((outs, pool.as_tensor().clone()))
    for a, b in zip(results[0][0], results[1][0]):
        assert torch.equal(a, b)
    assert torch.equal(results[0][1], results[1][1])


def test_attention_rejects_context_beyond_the_table(dev):
    """max_ctx larger than a block-table row could read past it: refused."""
    layout = LLAMA8B
    pool = kvx.Pool(8, layout.page_bytes(), device=0)
    att = kvx.Attention(layout, 32, 4)  # rows of 4 pages = 64 tokens
    tables = torch.zeros(1, 4, dtype=torch.int32, device=dev)
    q = torch.zeros(1, 32, 128, dtype=torch.bfloat16, device=dev)
    out = torch.empty(1, 32, 128, dtype=torch.float32, device=dev)
    ctx = torch.tensor([65], dtype=torch.int32, device=dev)
    with pytest.raises(kvx.KvxError):
        att(pool, tables, ctx, q, out, 1, 65)


def test_host_pool_zero_copy_roundtrip(dev):
    """DEVICE -> mapped pinned HOST pool -> DEVICE with the SM mover (PCIe)."""
    layout = TINY
    pb = layout.page_bytes()
    n = 24
    ids = np.arange(n, dtype=np.uint32)[::-1].copy()
    tags = O.tags_array(1, 0, np.arange(n))
    src, ref = filled_pool(layout, n, ids, tags, 11, kvx.FILL_BITS, dev)
    host = kvx.Pool(n, pb, host=True)
    back = kvx.Pool(n, pb, device=0)
    hid = to_dev(np.arange(n, dtype=np.int32), dev)
    kvx.copy_pages(src, to_dev(ids.view(np.int32), dev), host, hid, n, kvx.COPY_SM)
    kvx.copy_pages(host, hid, back, to_dev(ids.view(np.int32), dev), n, kvx.COPY_SM)
    torch.cuda.synchronize()
    assert np.array_equal(host.as_tensor().numpy(), ref[ids])
    assert np.array_equal(back.as_tensor().cpu().numpy(), ref)


@pytest.mark.parametrize("layout", [TINY, LLAMA8B], ids=["tiny-f32", "8b-bf16"])
def test_append_kv_bit_exact(dev, layout):
    pb = layout.page_bytes()
    rng = np.random.default_rng(3)
    n, pages = 9, 16
    ids = rng.permutation(pages)[:n].astype(np.uint32)
    slots = rng.integers(0, layout.block_tokens, n).astype(np.int32)
    elt = np.float32 if layout.dtype == kvx.F32 else np.uint16
    k = rng.integers(0, 2**15, (n, layout.num_kv_heads, layout.head_dim)).astype(elt)
    v = rng.integers(0, 2**15, (n, layout.num_kv_heads, layout.head_dim)).astype(elt)
    all_ids = np.arange(pages, dtype=np.uint32)
    pool, ref = filled_pool(layout, pages, all_ids, O.tags_array(0, 0, all_ids), 5, kvx.FILL_BITS, dev)
    kvx.append_kv(pool, layout, to_dev(ids.view(np.int32), dev), to_dev(slots, dev), to_dev(k, dev), to_dev(v, dev), n)
    O.append_kv(ref, olayout(layout), ids, slots, k, v)
    torch.cuda.synchronize()
    assert np.array_equal(pool.as_tensor().cpu().numpy(), ref)


def _attention_case(dev, layout, hq, ctx_lens, splits=0, seed=0, merge=kvx.MERGE_AUTO, flags=0):
    rng = np.random.default_rng(seed)
    pb = layout.page_bytes()
    batch = len(ctx_lens)
    max_ctx = int(max(ctx_lens))
    max_blocks = (max_ctx + layout.block_tokens - 1) // layout.block_tokens
    pages = batch * max_blocks + 5
    perm = rng.permutation(pages).astype(np.uint32)
    tables = perm[:batch * max_blocks].reshape(batch, max_blocks)
    all_ids = np.arange(pages, dtype=np.uint32)
    pool, ref = filled_pool(layout, pages, all_ids, O.tags_array(2, 1, all_ids), seed + 77, kvx.FILL_VALUES, dev)
    if layout.dtype == kvx.BF16:
        qf = rng.standard_normal((batch, hq, layout.head_dim)).astype(np.float32)
        q = (qf.view(np.uint32) + 0x7FFF + ((qf.view(np.uint32) >> 16) & 1) >> 16).astype(np.uint16)
    else:
        q = rng.standard_normal((batch, hq, layout.head_dim)).astype(np.float32)
    ctx = np.asarray(ctx_lens, np.int32)
    att = kvx.Attention(layout, hq, max_blocks, num_splits=splits, split_merge=merge, flags=flags)
    ws_bytes = att.workspace_bytes(batch, max_ctx)
    ws = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=dev) if ws_bytes else None
    out = torch.full((batch, hq, layout.head_dim), float("nan"), dtype=torch.float32, device=dev)
    att(pool, to_dev(tables.view(np.int32), dev), to_dev(ctx, dev), to_dev(q, dev), out, batch, max_ctx, ws)
    torch.cuda.synchronize()
    scale = 1.0 / np.sqrt(np.float32(layout.head_dim))
    expect = O.decode_attention(ref, olayout(layout), hq, tables, ctx, q, float(np.float32(scale)))
    return out.cpu().numpy().astype(np.float64), expect


@pytest.mark.parametrize("ctx_lens", [[384], [1, 17, 200, 384], [16, 33], [0, 17, 0]])
def test_attention_tiny_fp32(dev, ctx_lens):
    got, ref = _attention_case(dev, TINY, 8, ctx_lens)
    assert np.all(np.abs(got - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref))), np.abs(got - ref).max()


@pytest.mark.parametrize("merge", [kvx.MERGE_AUTO, kvx.MERGE_GLOBAL], ids=["auto", "global"])
@pytest.mark.parametrize("hq,ctx_lens,splits", [
    (32, [8192], 0), (32, [1, 15, 16, 17, 500, 1031], 0), (64, [4096, 33], 0), (8, [700], 1),
    (32, [3000, 2999, 64], 7), (128, [257], 0), (32, [8192] * 8, 0),
    (32, [0, 300, 0], 0), (32, [0, 4096], 5),  # empty requests (a session with no tokens yet) -> zeros
])
def test_attention_bf16_d128(dev, hq, ctx_lens, splits, merge):
    got, ref = _attention_case(dev, LLAMA8B, hq, ctx_lens, splits, seed=len(ctx_lens) + hq, merge=merge)
    err = np.abs(got - ref)
    assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), (err.max(), err.mean())
    assert err.mean() < 5e-4


@pytest.mark.parametrize("hq,ctx_lens,splits", [
    (32, [8192], 16), (32, [8192], 2), (32, [5000, 16], 9), (32, [100], 16), (64, [1, 2, 3, 4], 4),
    (4, [16 * 1024 * 16], 16), (32, [0, 5000, 0], 4),
])
def test_attention_cluster_merge(dev, hq, ctx_lens, splits):
    """Split-K partials merged over DSMEM inside a thread-block cluster
    (KVX_MERGE_CLUSTER): split counts up to 16, splits with no pages (ctx 100
    over 16 splits), and the longest context one cluster covers (16 splits x
    1,024 staged pages = 262,144 tokens, on a one-kv-head layout)."""
    layout = LLAMA8B if hq % 8 == 0 else kvx.PageLayout(1, 128, 16, kvx.BF16)
    got, ref = _attention_case(dev, layout, hq, ctx_lens, splits, seed=splits, merge=kvx.MERGE_CLUSTER)
    err = np.abs(got - ref)
    assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), (err.max(), err.mean())
    assert err.mean() < 5e-4


@pytest.mark.parametrize("hq,ctx_lens,splits,groups", [
    (32, [32768], 16, 4), (32, [8192], 12, 2), (32, [5000, 16, 0], 15, 3), (64, [4096], 8, 2),
    (32, [100], 16, 2),  # slices with no pages in some clusters
])
def test_attention_two_level_cluster_merge(dev, hq, ctx_lens, splits, groups):
    """KVX_ATTN_CLUSTERS(G): the splits of a (request, kv head) form G
    clusters of splits/G CTAs; each cluster merges over DSMEM, then the last
    owner of each output slice merges the G cluster results from the
    workspace. Checked against the fp64 oracle, twice in a row (the arrival
    counters reset)."""
    flags = kvx.ATTN_EARLY_PREFETCH | (groups << 8)
    for rep in range(2):
        got, ref = _attention_case(dev, LLAMA8B, hq, ctx_lens, splits, seed=splits + rep, merge=kvx.MERGE_AUTO,
                                   flags=flags)
        err = np.abs(got - ref)
        assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), (rep, err.max(), err.mean())
        assert err.mean() < 5e-4


def test_attention_cluster_merge_refuses_what_does_not_fit(dev):
    # 17 splits exceed the largest cluster; asking for CLUSTER must fail, not fall back silently
    with pytest.raises(kvx.KvxError, match="cluster"):
        _attention_case(dev, LLAMA8B, 32, [4096], 17, merge=kvx.MERGE_CLUSTER)


def test_full_session_migration_property(dev):
    """Config 2 at full size (1 GiB, 8B @ 8K): fill a session's 16,384 pages
    at a random permutation, pack every layer, unpack into a second
    permutation, and check every landed page equals a fresh fill of its tag."""
    layout = LLAMA8B
    pb = layout.page_bytes()
    L, blocks = 32, 512
    n = L * blocks
    rng = np.random.default_rng(2026)
    pool_pages = 2 * n
    src_ids = rng.permutation(pool_pages)[:n].astype(np.uint32)
    dst_ids = rng.permutation(pool_pages)[:n].astype(np.uint32)
    tags = O.tags_array(0, np.repeat(np.arange(L), blocks), np.tile(np.arange(blocks), L))
    src = kvx.Pool(pool_pages, pb)
    dst = kvx.Pool(pool_pages, pb)
    t_tags = to_dev(tags.view(np.int32), dev)
    kvx.fill_pages(src, to_dev(src_ids.view(np.int32), dev), t_tags, n, 123, layout, kvx.FILL_BITS)
    buf = torch.empty(blocks * pb, dtype=torch.uint8, device=dev)
    d_src, d_dst = to_dev(src_ids.view(np.int32), dev), to_dev(dst_ids.view(np.int32), dev)
    for l in range(L):
        sl = slice(l * blocks, (l + 1) * blocks)
        kvx.pack(src, d_src[sl], blocks, buf, kvx.COPY_TMA if l % 2 else kvx.COPY_SM)
        kvx.unpack(dst, d_dst[sl], blocks, buf, kvx.COPY_SM if l % 2 else kvx.COPY_TMA)
    expect = kvx.Pool(pool_pages, pb)
    kvx.fill_pages(expect, d_dst, t_tags, n, 123, layout, kvx.FILL_BITS)
    torch.cuda.synchronize()
    a, b = dst.as_tensor(), expect.as_tensor()
    idx = d_dst.long()
    assert torch.equal(a[idx], b[idx])


@pytest.mark.parametrize("merge", [kvx.MERGE_GLOBAL, kvx.MERGE_CLUSTER])
def test_attention_split_merge_reuses_workspace(dev, merge):
    """The in-kernel split merge leaves its arrival counters zeroed (global) /
    its cluster barriers re-armed (cluster): repeated launches give
    bit-identical results (static page deal, fixed merge order), for several
    split counts."""
    layout = LLAMA8B
    for splits in ((2, 5, 32) if merge == kvx.MERGE_GLOBAL else (2, 5, 6)):
        got0, ref = _attention_case(dev, layout, 32, [2048, 1500, 77], splits, seed=splits, merge=merge)
        err = np.abs(got0 - ref)
        assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), (splits, err.max())
    rng = np.random.default_rng(9)
    pb = layout.page_bytes()
    pages = 3 * 128
    all_ids = np.arange(pages, dtype=np.uint32)
    pool, _ = filled_pool(layout, pages, all_ids, O.tags_array(4, 4, all_ids), 3, kvx.FILL_VALUES, dev)
    tables = to_dev(rng.permutation(pages).astype(np.int32).reshape(3, 128), dev)
    ctx = to_dev(np.array([2048, 2000, 1], np.int32), dev)
    q = to_dev(rng.integers(0x3C00, 0x3F80, (3, 32, 128)).astype(np.uint16), dev)
    att = kvx.Attention(layout, 32, 128, num_splits=7 if merge == kvx.MERGE_GLOBAL else 5, split_merge=merge)
    ws = torch.zeros(att.workspace_bytes(3, 2048), dtype=torch.uint8, device=dev)
    outs = []
    for _ in range(4):
        out = torch.empty(3, 32, 128, dtype=torch.float32, device=dev)
        att(pool, tables, ctx, q, out, 3, 2048, ws)
        outs.append(out)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("layout,hq,splits", [(LLAMA8B, 32, 0), (LLAMA8B, 32, 5), (LLAMA8B, 64, 3), (TINY, 8, 0)],
                         ids=["8b-auto", "8b-5splits", "70b-3splits", "tiny-f32"])
def test_fused_append_decode_step(dev, layout, hq, splits):
    """kvx_decode_attention_append (append this step's K/V at ctx-1, then
    attend) == kvx_append_kv + kvx_decode_attention: identical pool bytes
    and bit-identical outputs; lengths at page boundaries (ctx % 16 in
    {1, 0, 15}) and a one-token request."""
    pb = layout.page_bytes()
    rng = np.random.default_rng(hq + splits)
    ctx_lens = np.array([1, 16, 17, 31, 500, 1024], np.int32)
    B = len(ctx_lens)
    mb = 64
    pages = B * mb + 3
    all_ids = np.arange(pages, dtype=np.uint32)
    tables = rng.permutation(pages)[:B * mb].astype(np.uint32).reshape(B, mb)
    pool_a, _ = filled_pool(layout, pages, all_ids, O.tags_array(6, 1, all_ids), 31, kvx.FILL_VALUES, dev)
    pool_b, _ = filled_pool(layout, pages, all_ids, O.tags_array(6, 1, all_ids), 31, kvx.FILL_VALUES, dev)
    elt = torch.bfloat16 if layout.dtype == kvx.BF16 else torch.float32
    H, D = layout.num_kv_heads, layout.head_dim
    nk = torch.randn(B, H, D, device=dev).to(elt)
    nv = torch.randn(B, H, D, device=dev).to(elt)
    q = torch.randn(B, hq, D, device=dev).to(elt)
    d_tables, d_ctx = to_dev(tables.view(np.int32), dev), to_dev(ctx_lens, dev)
    att = kvx.Attention(layout, hq, mb, num_splits=splits)
    ws = torch.zeros(max(att.workspace_bytes(B, mb * 16), 1), dtype=torch.uint8, device=dev)
    out_a = torch.empty(B, hq, D, dtype=torch.float32, device=dev)
    out_b = torch.empty_like(out_a)
    att(pool_a, d_tables, d_ctx, q, out_a, B, mb * 16, ws, new_k=nk, new_v=nv)
    t = ctx_lens - 1
    ids = to_dev(tables[np.arange(B), t // 16].astype(np.int32), dev)
    kvx.append_kv(pool_b, layout, ids, to_dev((t % 16).astype(np.int32), dev), nk, nv, B)
    att(pool_b, d_tables, d_ctx, q, out_b, B, mb * 16, ws)
    torch.cuda.synchronize()
    assert torch.equal(pool_a.as_tensor(), pool_b.as_tensor())
    assert torch.equal(out_a, out_b)
    # and against the fp64 oracle over the pool the fused step left behind
    _check_against_oracle(pool_a, layout, hq, tables, ctx_lens, q, out_a)


def _check_against_oracle(pool, layout, hq, tables, ctx_lens, q, out):
    qn = q.cpu().view(torch.int16).numpy().view(np.uint16) if q.dtype == torch.bfloat16 else q.cpu().numpy()
    scale = float(np.float32(1.0 / np.sqrt(np.float32(layout.head_dim))))
    ref = O.decode_attention(pool.as_tensor().cpu().numpy(), olayout(layout), hq, tables, ctx_lens, qn, scale)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    if layout.dtype == kvx.BF16:
        assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), (err.max(), err.mean())
        assert err.mean() < 5e-4
    else:
        assert np.all(err <= 1e-5 * np.maximum(1.0, np.abs(ref))), err.max()


def test_fused_decode_step_full_size(dev):
    """Config 2's decode shape at full context (8B KV, ctx 8192, batch 4,
    auto plan = clustered split-K): the fused step equals append + attention
    bit for bit, and the appended rows are where the block table says."""
    layout = LLAMA8B
    pb = layout.page_bytes()
    B, ctx, mb = 4, 8192, 512
    pages = B * mb
    rng = np.random.default_rng(77)
    tables = rng.permutation(pages).astype(np.uint32).reshape(B, mb)
    ids = torch.arange(pages, dtype=torch.int32, device=dev)
    tags = torch.stack([ids * 0 + 9, ids * 0, ids], -1).contiguous()
    pool_a = kvx.Pool(pages, pb, device=0)
    pool_b = kvx.Pool(pages, pb, device=0)
    for p_ in (pool_a, pool_b):
        kvx.fill_pages(p_, ids, tags, pages, 5, layout, kvx.FILL_VALUES)
    nk = torch.randn(B, 8, 128, device=dev).to(torch.bfloat16)
    nv = torch.randn(B, 8, 128, device=dev).to(torch.bfloat16)
    q = torch.randn(B, 32, 128, device=dev).to(torch.bfloat16)
    lens = np.array([ctx, ctx - 15, ctx - 16, 4097], np.int32)
    d_tables, d_ctx = to_dev(tables.view(np.int32), dev), to_dev(lens, dev)
    att = kvx.Attention(layout, 32, mb)
    ws = torch.zeros(max(att.workspace_bytes(B, ctx), 1), dtype=torch.uint8, device=dev)
    out_a = torch.empty(B, 32, 128, dtype=torch.float32, device=dev)
    out_b = torch.empty_like(out_a)
    att(pool_a, d_tables, d_ctx, q, out_a, B, ctx, ws, new_k=nk, new_v=nv)
    t = lens - 1
    kvx.append_kv(pool_b, layout, to_dev(tables[np.arange(B), t // 16].astype(np.int32), dev),
                  to_dev((t % 16).astype(np.int32), dev), nk, nv, B)
    att(pool_b, d_tables, d_ctx, q, out_b, B, ctx, ws)
    torch.cuda.synchronize()
    assert torch.equal(pool_a.as_tensor(), pool_b.as_tensor())
    assert torch.equal(out_a, out_b)
    _check_against_oracle(pool_a, layout, 32, tables, lens, q, out_a)
    page = pool_a.as_tensor()[int(tables[1, t[1] // 16])].view(torch.bfloat16).view(2, 8, 16, 128)
    assert torch.equal(page[0, :, t[1] % 16], nk[1]) and torch.equal(page[1, :, t[1] % 16], nv[1])


def test_full_70b_session_migration_property(dev):
    """Config 3 at full size on one GPU (10.7 GB, Llama-3.1-70B KV @ 32K):
    every layer's 2,048 pages move page->page (K3, the migration kernel) into
    a second pool standing in for the receiver; every landed page must equal a
    fresh fill of its (session, layer, block) tag."""
    layout = LLAMA8B  # 70B KV page shape is the same: 8 kv heads x d128 bf16
    pb = layout.page_bytes()
    L, blocks = 80, 2048
    n = L * blocks
    if torch.cuda.get_device_properties(0).total_memory < 4 * n * pb:
        pytest.skip("needs ~43 GB of device memory")
    gen = torch.Generator(device="cpu").manual_seed(70)
    src_ids = torch.randperm(n + 1000, generator=gen)[:n].to(torch.int32).to(dev)
    dst_ids = torch.randperm(n + 1000, generator=gen)[:n].to(torch.int32).to(dev)
    layer = torch.arange(L, dtype=torch.int32).repeat_interleave(blocks)
    block = torch.arange(blocks, dtype=torch.int32).repeat(L)
    tags = torch.stack([torch.full_like(layer, 70), layer, block], -1).contiguous().to(dev)
    src = kvx.Pool(n + 1000, pb)
    dst = kvx.Pool(n + 1000, pb)
    kvx.fill_pages(src, src_ids, tags, n, 700, layout, kvx.FILL_BITS)
    for l in range(L):
        sl = slice(l * blocks, (l + 1) * blocks)
        kvx.copy_pages(src, src_ids[sl], dst, dst_ids[sl], blocks, kvx.COPY_AUTO)
    del src
    expect = kvx.Pool(n, pb)
    kvx.fill_pages(expect, torch.arange(n, dtype=torch.int32, device=dev), tags, n, 700, layout, kvx.FILL_BITS)
    torch.cuda.synchronize()
    got, want = dst.as_tensor(), expect.as_tensor()
    for l in range(0, L, 8):  # compare in chunks to bound temporary memory
        sl = slice(l * blocks, min(L, l + 8) * blocks)
        assert torch.equal(got[dst_ids[sl].long()], want[sl])


def test_corrupt_page_id_fails_loudly(dev, tmp_path):
    """An out-of-range page id in a block table traps the kernel (no silent
    out-of-bounds copy); run in a child process since a trap poisons the
    CUDA context."""
    import subprocess
    import sys
    script = tmp_path / "bad_id.py"
    script.write_text(
        "import sys, torch\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "from paper_2412_16434_b200 import kvx\n"
        "pool = kvx.Pool(8, 4096)\n"
        "ids = torch.tensor([1, 99], dtype=torch.int32, device='cuda')\n"
        "buf = torch.empty(2 * 4096, dtype=torch.uint8, device='cuda')\n"
        "try:\n"
        "    kvx.pack(pool, ids, 2, buf, kvx.COPY_SM)\n"
        "    torch.cuda.synchronize()\n"
        "except Exception as e:\n"
        "    print('raised', type(e).__name__)\n"
        "    sys.exit(0)\n"
        "sys.exit(3)\n")
    proc = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0 and "raised" in proc.stdout, proc.stdout + proc.stderr[-2000:]
