"""Physical payload behind the store, on the B200 (lockstep and free-running).

A KvStore with a NodePayload attached gives every tier copy a real page; the
transfers the state machine schedules move real bytes when they are applied
in (complete_at, id) order — the contract of the reference's test drivers
(Pump, /root/reference/proj/tests/test_kvstore.cpp:24-41). After every step
we check, for every block of every session:
  * each residency bit the store reports has exactly one physical copy, in the
    pool the tier maps to (DEVICE -> HBM pool; HOST -> pinned host pool, or the
    HBM landing pool for migrated blocks; DISK -> disk pool), and no pool
    holds a page the store does not account for (no leaks);
  * every copy's bytes equal the block's content as created (bit-exact
    against the CPU oracle's fill of the same (session, layer, block) tag).
"""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2412_16434_b200 import kvstore as K  # noqa: E402

import oracle.oracle as O  # noqa: E402  (test infrastructure)

SEED = 0x5EED
LAYERS = 2


def tiny_profile():
    # config 1 shape: 2 layers x 4 kv heads x d64 fp32 -> 32 KiB pages
    return K.GpuProfile(kv_bytes_per_token=LAYERS * 2 * 4 * 64 * 4, num_layers=LAYERS, hbm_capacity=10**12)


_DISK = {"dir": None, "n": 0}


@pytest.fixture(params=["disk-pinned", "disk-file"], autouse=True)
def disk_backing(request, tmp_path):
    """Every test runs twice: DISK tier in pinned host memory, and DISK tier
    in files (kvx_pool_create_file: preads / pwrites in stream order, HBM
    <-> file through the per-lane bounce pages)."""
    _DISK["dir"] = tmp_path if request.param == "disk-file" else None
    yield
    _DISK["dir"] = None


def payload_opts(device_pages=64, host_pages=64, landing_pages=64, disk_pages=128, free_running=False):
    path = ""
    if _DISK["dir"] is not None:
        _DISK["n"] += 1
        path = str(_DISK["dir"] / f"disk{_DISK['n']}.pages")
    return K.PayloadOptions(device=0, num_kv_heads=4, head_dim=64, block_tokens=16, dtype=0, fill_mode=1,
                            device_pages=device_pages, host_pages=host_pages, landing_pages=landing_pages,
                            disk_pages=disk_pages, seed=SEED, free_running=free_running, disk_path=path)


MODES = pytest.mark.parametrize("free_running", [False, True], ids=["lockstep", "free-running"])


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0


_EXPECT = {}


def expected(session, layer, block, pb):
    key = (session, layer, block)
    if key not in _EXPECT:
        buf = np.zeros((1, pb), np.uint8)
        O.fill_pages(buf, pb, np.zeros(1, np.uint32), O.tags_array(session, layer, block), SEED,
                     O.Layout(4, 64, 16, 0), 1)
        _EXPECT[key] = buf[0]
    return _EXPECT[key]


def verify(store, node, sessions, landing_ok=True):
    pb = store.layer_block_bytes()
    held = [0, 0, 0, 0]
    for s in sessions:
        span = (store.cached_tokens(s) + 15) // 16 + 4  # a few past the table too
        for l in range(LAYERS):
            for b in range(max(span, 8)):
                r = store.residency(s, l, b)
                for t in range(3):
                    pool = node.pool_of(s, l, b, t)
                    if r & (1 << t):
                        assert pool >= 0, f"s{s} l{l} b{b}: tier {t} resident but no page"
                        if t == K.DEVICE:
                            assert pool == K.POOL_DEVICE
                        elif t == K.HOST:
                            assert pool in (K.POOL_HOST, K.POOL_LANDING) and (landing_ok or pool == K.POOL_HOST)
                        else:
                            assert pool == K.POOL_DISK
                        held[pool] += 1
                        got = node.read_block(s, l, b, t, pb)
                        assert np.array_equal(got, expected(s, l, b, pb)), f"s{s} l{l} b{b} tier {t}: bytes differ"
                    else:
                        assert pool < 0, f"s{s} l{l} b{b}: tier {t} not resident but holds a page"
    in_flight = node.stats()["in_flight"]  # free-running: moves issued, not yet applied
    for p in range(4):
        assert node.pages_in_use(p) == held[p] + in_flight[p], \
            f"pool {p}: {node.pages_in_use(p)} pages in use, {held[p]} resident + {in_flight[p]} in flight"


class Pump:
    def __init__(self, store):
        self.store, self.pending = store, []

    def add(self, sched):
        self.pending += list(sched)

    def run(self, limit=None):
        self.pending.sort(key=lambda t: (t[1], t[0]))
        todo = self.pending if limit is None else self.pending[:limit]
        out = [self.store.apply_transfer(tid, at) for tid, at in todo]
        self.pending = self.pending[len(todo):]
        return out


def make_node(opts_kw=None, free_running=False, **store_kw):
    cluster = K.PayloadCluster()
    store = K.KvStore(gpu=tiny_profile(), opts=K.Options(**store_kw))
    node = K.NodePayload(cluster, store_kw.get("node_id", 0),
                         payload_opts(free_running=free_running, **(opts_kw or {})))
    node.attach(store)
    return cluster, store, node


@MODES
def test_write_behind_purge_reload(dev, free_running):
    cluster, store, node = make_node(free_running=free_running)
    pump = Pump(store)
    for s in (1, 2):
        store.register_session(s, f"s{s}")
    store.finalize_sessions()
    keys, sched = store.append_blocks(1, 40, 0)  # 3 blocks per layer
    pump.add(sched)
    verify(store, node, [1, 2])
    pump.run()
    verify(store, node, [1, 2])
    assert node.pages_in_use(K.POOL_HOST) == 6 and node.pages_in_use(K.POOL_DISK) == 6
    freed, sched = store.purge_from_device(store.layer_block_bytes() * 6, 1_000_000, False)
    assert freed == store.layer_block_bytes() * 6 and not sched
    verify(store, node, [1, 2])
    assert node.pages_in_use(K.POOL_DEVICE) == 0
    plan, sched = store.plan_layerwise_load(1, 2_000_000, 100_000, K.DEMAND)
    pump.add(sched)
    pump.run()
    assert store.fully_device_resident(1)
    verify(store, node, [1, 2])
    moved = node.bytes_moved()
    assert moved["load_h2d"] == 6 * store.layer_block_bytes()
    store.release_session(1, 3_000_000)
    verify(store, node, [1, 2])
    assert sum(node.pages_in_use(p) for p in range(4)) == 0


@MODES
def test_swap_offload_and_reactivation(dev, free_running):
    cluster, store, node = make_node(free_running=free_running, write_behind=False)
    pump = Pump(store)
    store.register_session(1, "a")
    store.register_session(2, "b")
    store.finalize_sessions()
    pump.add(store.append_blocks(1, 33, 0)[1])
    pump.add(store.append_blocks(2, 16, 0)[1])
    pump.add(store.offload_session(1, 10))
    verify(store, node, [1, 2])
    pump.run(limit=2)
    verify(store, node, [1, 2])
    store.set_active(1, True, 20)  # voids the rest of the offload
    pump.run()
    verify(store, node, [1, 2])
    pump.add(store.offload_session(2, 30))
    pump.run()
    verify(store, node, [1, 2])
    assert not store.fully_device_resident(2) and store.has_any_copy(2)


@MODES
@pytest.mark.parametrize("cap", [0, 2], ids=["uncapped", "capped-2-ctas"])
def test_migration_lands_in_receiver_hbm(dev, free_running, cap):
    """import_migration on node 1 pulls the frozen session from node 0: each
    layer's NetArrive lands in node 1's HBM landing pool (HOST tier in the
    ledger, reference kvstore.cpp:914-923); the follow-up demand load is an
    HBM->HBM page copy. Also with the migration pushes' grid capped
    (PayloadOptions.migrate_max_ctas)."""
    cluster = K.PayloadCluster()
    stores, nodes, pumps = [], [], []
    for n in range(2):
        st = K.KvStore(gpu=tiny_profile(), opts=K.Options(node_id=n))
        opts = payload_opts(free_running=free_running)
        opts.migrate_max_ctas = cap
        nd = K.NodePayload(cluster, n, opts)
        nd.attach(st)
        st.register_session(5, "mig")
        st.finalize_sessions()
        stores.append(st), nodes.append(nd), pumps.append(Pump(st))
    pumps[0].add(stores[0].append_blocks(5, 70, 0)[1])
    pumps[0].run()
    stores[0].mark_migrating_out(5)
    pumps[1].add(stores[1].import_migration(5, stores[0].cached_tokens(5), 1_000_000))
    res = pumps[1].run()
    assert sum(r.migration_complete for r in res) == 1
    for l in range(LAYERS):
        for b in range(5):
            assert nodes[1].pool_of(5, l, b, K.HOST) == K.POOL_LANDING
    verify(stores[1], nodes[1], [5])
    stores[0].release_session(5, 2_000_000)
    verify(stores[0], nodes[0], [5])
    assert sum(nodes[0].pages_in_use(p) for p in range(4)) == 0
    plan, sched = stores[1].plan_layerwise_load(5, 3_000_000, 10_000, K.DEMAND)
    pumps[1].add(sched)
    pumps[1].run()
    assert stores[1].fully_device_resident(5)
    verify(stores[1], nodes[1], [5])
    assert nodes[1].bytes_moved()["net_arrive"] == 2 * 5 * stores[1].layer_block_bytes()


@MODES
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("write_behind", [True, False])
def test_randomized_lifecycle_keeps_bytes_and_state_consistent(dev, seed, write_behind, free_running):
    rng = random.Random(seed * 7 + write_behind)
    pb = 2 * 4 * 16 * 64 * 4
    cluster, store, node = make_node(opts_kw=dict(device_pages=96, host_pages=96, disk_pages=400),
                                     free_running=free_running,
                                     write_behind=write_behind, device_capacity=pb * 2 * 24,
                                     host_capacity=pb * 2 * 20)
    pump = Pump(store)
    sessions = [1, 2, 3]
    for s in sessions:
        store.register_session(s, f"id{s}", rng.random() < 0.3)
    store.finalize_sessions()
    now = 0
    for op in range(120):
        now += rng.randint(0, 300_000)
        s = rng.choice(sessions)
        kind = rng.randint(0, 9)
        try:
            if kind <= 2:
                need = store.bytes_for_new_blocks(s, rng.randint(1, 20))
                if need <= store.device_free():
                    pump.add(store.append_blocks(s, rng.randint(1, 20), now)[1])
            elif kind == 3:
                pump.add(store.purge_from_device(pb * rng.randint(1, 6), now, rng.random() < 0.5)[1])
            elif kind == 4:
                plan, sched = store.plan_layerwise_load(s, now, 50_000, K.DEMAND)
                pump.add(sched)
            elif kind == 5:
                pump.add(store.promote(s, now)[1])
            elif kind == 6:
                pump.add(store.offload_session(s, now))
            elif kind == 7:
                store.set_active(s, rng.random() < 0.5, now)
            elif kind == 8 and rng.random() < 0.2:
                store.release_session(s, now)
            else:
                pump.run(limit=rng.randint(1, 5))
        except (K.KvsLogicError, K.KvsRuntimeError) as e:
            # contract violations the reference also raises (e.g. loading a
            # block whose only copy was dropped); payload errors would fail here
            assert "payload" not in str(e), e
        if op % 10 == 0:
            verify(store, node, sessions)
    pump.run()
    verify(store, node, sessions)


def test_recycled_pages_wait_for_other_lanes(dev):
    """Free-running, pages recycled across lanes: session A's write-behind
    DiskWrites (DISK lane) still read A's DEVICE pages when A is purged from
    DEVICE (its HOST copy has landed, on the OUT lane) and B's demand load (IN
    lane) is handed those very pages. The DISK lane is stalled by a 50 ms spin
    kernel queued ahead of A's writes, so without the page fences B's load
    would overwrite the pages before the DiskWrites read them and A's DISK
    copy would hold B's bytes. The freed pages stay quarantined until the
    DiskWrite batch completes, so the load's allocation must wait for it
    (counted in cross_lane_waits), and every copy of both sessions stays
    bit-exact."""
    cluster, store, node = make_node(opts_kw=dict(device_pages=6), free_running=True)
    pump = Pump(store)
    for s in (1, 2):
        store.register_session(s, f"s{s}")
    store.finalize_sessions()
    pump.add(store.append_blocks(2, 40, 0)[1])  # B: 3 blocks x 2 layers fill the 6-page pool
    pump.run()
    freed, _ = store.purge_from_device(store.layer_block_bytes() * 6, 1_000_000, False)
    assert freed == store.layer_block_bytes() * 6
    node.synchronize()
    with torch.cuda.stream(torch.cuda.ExternalStream(node.stream(K.LANE_DISK))):
        torch.cuda._sleep(100_000_000)  # ~50 ms at B200 clocks
    pump.add(store.append_blocks(1, 40, 2_000_000)[1])  # A reuses B's pages; HostCopy + DiskWrite posted
    pump.run(limit=LAYERS)  # A's HOST copies land (OUT lane); the DiskWrites wait behind the spin
    assert pump.pending, "the DiskWrites must still be pending"
    freed, _ = store.purge_from_device(store.layer_block_bytes() * 6, 3_000_000, False)
    assert freed == store.layer_block_bytes() * 6 and node.pages_in_use(K.POOL_DEVICE) == 0
    before = node.stats()["cross_lane_waits"]
    plan, sched = store.plan_layerwise_load(2, 4_000_000, 100_000, K.DEMAND)
    assert plan.any_load
    assert node.stats()["cross_lane_waits"] > before, "the load did not wait for the DiskWrites reading its pages"
    pump.add(sched)
    pump.run()
    assert store.fully_device_resident(2)
    verify(store, node, [1, 2])
