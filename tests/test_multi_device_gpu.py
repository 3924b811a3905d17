"""Two payload nodes on two GPUs in one process (PayloadCluster, node i on
cuda:i): a session migrated through the store API lands in the receiver
GPU's landing pool over peer access (NVLink on an HGX box), bit-exact, and
is then loaded into the receiver's DEVICE pages. Skips on a one-GPU box."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2412_16434_b200 import kvstore as K  # noqa: E402
from paper_2412_16434_b200 import kvx  # noqa: E402

import oracle.oracle as O  # noqa: E402  (test infrastructure)

LAYERS, HEADS, DIM, SEED, TOKENS = 4, 8, 128, 0x2D, 1000


@pytest.mark.parametrize("free_running", [False, True], ids=["lockstep", "free-running"])
def test_migration_between_two_gpus(free_running):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    gpu = K.GpuProfile(kv_bytes_per_token=LAYERS * 2 * HEADS * DIM * 2, num_layers=LAYERS, hbm_capacity=10**12)
    cluster = K.PayloadCluster()
    stores, nodes = [], []
    for n in range(2):
        st = K.KvStore(gpu=gpu, opts=K.Options(node_id=n))
        nd = K.NodePayload(cluster, n, K.PayloadOptions(device=n, num_kv_heads=HEADS, head_dim=DIM, dtype=kvx.BF16,
                                                        device_pages=512, host_pages=512, landing_pages=512,
                                                        disk_pages=512, seed=SEED, free_running=free_running))
        nd.attach(st)
        st.register_session(1, "two-gpu")
        st.finalize_sessions()
        stores.append(st)
        nodes.append(nd)

    def pump(store, sched):
        for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
            store.apply_transfer(tid, at)

    _, sched = stores[0].append_blocks(1, TOKENS, 0)
    pump(stores[0], sched)
    stores[0].mark_migrating_out(1)
    pump(stores[1], stores[1].import_migration(1, TOKENS, 10_000_000))
    stores[0].release_session(1, 20_000_000)
    _, sched = stores[1].plan_layerwise_load(1, 30_000_000, 10_000, K.DEMAND)
    pump(stores[1], sched)
    assert stores[1].fully_device_resident(1)
    pb = 2 * HEADS * 16 * DIM * 2
    blocks = (TOKENS + 15) // 16
    for layer in range(LAYERS):
        for b in (0, blocks // 2, blocks - 1):
            want = np.zeros((1, pb), np.uint8)
            O.fill_pages(want, pb, np.zeros(1, np.uint32), O.tags_array(1, layer, b), SEED, O.Layout(HEADS, DIM, 16, 1), 1)
            assert np.array_equal(nodes[1].read_block(1, layer, b, K.DEVICE, pb), want[0]), (layer, b)
    assert nodes[1].bytes_moved()["net_arrive"] == LAYERS * blocks * pb
