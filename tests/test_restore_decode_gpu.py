"""Migrate, restore and consume: the whole hot path through the store API.

Node 0 holds a Llama-3.1-8B-shaped session (bf16, 16-token pages) created by
append_blocks; the store migrates it to node 1 (import_migration: per-layer
NetArrive into node 1's HBM landing pool via K3), releases the source, and
restores it to DEVICE with a layer-wise demand load (plan_layerwise_load,
reference kvstore.cpp:433-543) — with the payload free-running, every move is
issued when scheduled and completed at apply. Then K4 decodes over the pages
node 1 now holds, using the block-table rows the payload reports; the output
must match the CPU oracle's fp64 attention over the blocks' contents
(attention tolerance as in test_kvx_gpu.py).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2412_16434_b200 import kvstore as K  # noqa: E402
from paper_2412_16434_b200 import kvx  # noqa: E402

import oracle.oracle as O  # noqa: E402  (test infrastructure)

LAYERS, HEADS, DIM, SEED = 4, 8, 128, 0xABC


def pump(store, sched):
    for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
        store.apply_transfer(tid, at)


@pytest.mark.parametrize("free_running", [False, True], ids=["lockstep", "free-running"])
@pytest.mark.parametrize("tokens", [1000, 257])
def test_migrate_restore_then_decode(free_running, tokens):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gpu = K.GpuProfile(kv_bytes_per_token=LAYERS * 2 * HEADS * DIM * 2, num_layers=LAYERS, hbm_capacity=10**12)
    cluster = K.PayloadCluster()
    stores, nodes = [], []
    for n in range(2):
        st = K.KvStore(gpu=gpu, opts=K.Options(node_id=n))
        nd = K.NodePayload(cluster, n, K.PayloadOptions(device=0, num_kv_heads=HEADS, head_dim=DIM, dtype=kvx.BF16,
                                                        device_pages=512, host_pages=512, landing_pages=512,
                                                        disk_pages=512, seed=SEED, free_running=free_running))
        nd.attach(st)
        st.register_session(3, "restored")
        st.finalize_sessions()
        stores.append(st)
        nodes.append(nd)
    _, sched = stores[0].append_blocks(3, tokens, 0)
    pump(stores[0], sched)
    stores[0].mark_migrating_out(3)
    pump(stores[1], stores[1].import_migration(3, tokens, 10_000_000))
    stores[0].release_session(3, 20_000_000)
    plan, sched = stores[1].plan_layerwise_load(3, 30_000_000, 10_000, K.DEMAND)
    assert plan.any_load
    pump(stores[1], sched)
    assert stores[1].fully_device_resident(3)
    nodes[1].synchronize()

    blocks = (tokens + 15) // 16
    pb = 2 * HEADS * 16 * DIM * 2
    layout = kvx.PageLayout(HEADS, DIM, 16, kvx.BF16)
    pool = kvx.Pool.borrow(nodes[1].pool_handle(K.POOL_DEVICE), 512, pb)
    rng = np.random.default_rng(tokens)
    dev = torch.device("cuda:0")
    for layer in range(LAYERS):
        table = nodes[1].device_block_table(3, layer, blocks).reshape(1, blocks)
        q = rng.integers(0x3C00, 0x3F80, (1, 32, DIM)).astype(np.uint16)
        q[..., 1::2] ^= 0x8000
        att = kvx.Attention(layout, 32, blocks)
        ws = torch.zeros(max(att.workspace_bytes(1, tokens), 1), dtype=torch.uint8, device=dev)
        out = torch.empty(1, 32, DIM, dtype=torch.float32, device=dev)
        att(pool, torch.from_numpy(table.view(np.int32)).to(dev), torch.tensor([tokens], dtype=torch.int32, device=dev),
            torch.from_numpy(q).to(dev), out, 1, tokens, ws)
        torch.cuda.synchronize()
        # oracle: the blocks' contents as created on node 0, gathered in order
        ref_pool = np.zeros((blocks, pb), np.uint8)
        O.fill_pages(ref_pool, pb, np.arange(blocks, dtype=np.uint32), O.tags_array(3, layer, np.arange(blocks)),
                     SEED, O.Layout(HEADS, DIM, 16, 1), 1)
        expect = O.decode_attention(ref_pool, O.Layout(HEADS, DIM, 16, 1), 32,
                                    np.arange(blocks, dtype=np.uint32).reshape(1, blocks),
                                    np.array([tokens], np.int32), q, float(np.float32(1 / np.sqrt(np.float32(DIM)))))
        err = np.abs(out.cpu().numpy() - expect)
        assert np.all(err <= 2e-3 + 1e-2 * np.abs(expect)), (layer, err.max())
    assert nodes[1].bytes_moved()["net_arrive"] == LAYERS * blocks * pb
    assert nodes[1].bytes_moved()["load_h2d"] == LAYERS * blocks * pb
