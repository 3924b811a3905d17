#!/usr/bin/env python
"""bench.py — KV migration hot path on B200 (Symphony, arXiv 2412.16434).

Metric (BASELINE.json, verbatim): "KV migrate GB/s (% HBM/NVLink roofline);
requests/s at equal p50 latency". `value` = session KV bytes relocated per
second, whole job (each byte of the session counted once; GB = 1e9 B); the
roofline fraction is the `roofline` object; requests/s at equal p50 comes
from the calibrated serving sweeps in profiles/.

N=1 (config 2, Llama-3.1-8B KV shape @ 8K: 32 layers x 512 pages x 64 KiB =
1 GiB): one step packs every page of the session (K1, gather by block table
into the contiguous migration buffer) and unpacks it into a second page
permutation (K2) — the device half of a layer-wise migration. Inputs are
1 GiB, larger than the 126 MB L2, so no flush is needed between steps.
Also reported: the fused page->page mover (K3), the other mover variant,
paged decode attention (K4: 8B @8K batch 1/8/64, 70B @32K batch 1/4, the
fused decode step), migration beside decode, the DISK tier as files, `e2e`
through the store's own API — the reference arm's own operation, a session
migration: mark_migrating_out -> import_migration -> apply every NetArrive
(K3 push into the receiver's landing pool) -> release, block tables up and a
probe page down inside the timed region — with Symphony's HOST<->HBM swap
and the raw kvx round trip in `detail`, and the CPU restatement on the host
cores.

N>1 (config 3, Llama-3.1-70B KV shape @ 32K, ~10.7 GB per session):
migration-plus-serving. Every rank decodes a batch of 70B @32K requests on
its main stream while its own session migrates to rank (r+1) % N on a side
stream, the K3 kernel storing straight into the peer's page pool over NVLink
(CUDA IPC) — a point-to-point exchange, no collective; weak scaling. Also the
layer-wise pipeline gate across GPUs (device-side flags) and a HOST-tier to
HOST-tier e2e. `--migrate-mode nccl` swaps in pack + ncclSend/ncclRecv +
unpack for comparison.

`--impl reference` times the reference's CPU path on the host cores: the
reference KvStore's migration bookkeeping (oracle/_ref, 1 thread, as the
reference is single-threaded) plus the payload restatement (oracle/, OpenMP on
all cores) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json's metric, verbatim. `value` is its first half (KV migrate
# GB/s; the roofline fraction is the `roofline` object); the second half
# (requests/s at equal p50 latency) comes from the calibrated serving sweeps
# in profiles/ (tools/serving_equal_p50.py), not from a per-run measurement.
METRIC = "KV migrate GB/s (% HBM/NVLink roofline); requests/s at equal p50 latency"
UNIT = "GB/s"
GB = 1e9

# Shapes.
CFG_8B = dict(model="llama-3.1-8b-kv", layers=32, kv_heads=8, head_dim=128, block_tokens=16, ctx=8192)
CFG_70B = dict(model="llama-3.1-70b-kv", layers=80, kv_heads=8, head_dim=128, block_tokens=16, ctx=32768)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# NVLink denominators. MEASURED_PEAKS.json (driver-written) carries no NVLink
# figure; the profiling guide's measured peer copy (770 GB/s per direction on
# this pool, /opt/skills/guides/B200_PROFILING.md) is the roofline
# denominator, the north star's nominal 900 GB/s the second one.
NVLINK_PEAK_GBS = 770.0
NVLINK_NOMINAL_GBS = 900.0
NVLINK_PEAK_PROVENANCE = ("measured peer copy per direction, B200_PROFILING.md (not in MEASURED_PEAKS.json); "
                          "nominal 900 GB/s per direction reported beside it")


def DECODE_FLAGS(kvx):  # noqa: N802 — a constant that needs the loaded module
    """Every decode launch here keeps the decode-step contract of
    KVX_ATTN_EARLY_PREFETCH (include/kvx.h): the kernel before it in the
    stream writes no block table, no ctx_lens and no page but the one holding
    position ctx-1, so tables and first pages are fetched before the PDL wait."""
    return kvx.ATTN_EARLY_PREFETCH


class ClockSampler:
    """NVML sampler thread: SM clock and clock-event reasons during timing."""

    NAMES = {
        "nvmlClocksEventReasonGpuIdle": "gpu_idle",
        "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks_setting",
        "nvmlClocksEventReasonSwPowerCap": "sw_power_cap",
        "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
        "nvmlClocksEventReasonSyncBoost": "sync_boost",
        "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
        "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
        "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake_slowdown",
    }

    def __init__(self, device_index: int, period_s: float = 0.01):
        self.period = period_s
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join()

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"], "samples": 0}
        reasons = [name for attr, name in self.NAMES.items()
                   if hasattr(self.nv, attr) and self.reasons & getattr(self.nv, attr)]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


def ncu_traffic(kernel: str):
    """Per-launch DRAM bytes from a committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# B200 arm


def session_pages(cfg):
    blocks = (cfg["ctx"] + cfg["block_tokens"] - 1) // cfg["block_tokens"]
    return blocks, cfg["layers"] * blocks


def make_session(torch, kvx, np, cfg, seed, dev, pool_pages=None, fill=True):
    """A pool holding one session's pages at a seeded random permutation."""
    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    pb = layout.page_bytes()
    blocks, n = session_pages(cfg)
    pool_pages = pool_pages or 2 * n
    rng = np.random.default_rng(seed)
    perm = rng.permutation(pool_pages).astype(np.uint32)
    src_ids, dst_ids = perm[:n], perm[n:2 * n] if pool_pages >= 2 * n else perm[:n]
    pool = kvx.Pool(pool_pages, pb, device=dev.index)
    d_src = torch.from_numpy(src_ids.view(np.int32)).to(dev)
    d_dst = torch.from_numpy(dst_ids.view(np.int32)).to(dev)
    if fill:
        layer = np.repeat(np.arange(cfg["layers"], dtype=np.uint32), blocks)
        block = np.tile(np.arange(blocks, dtype=np.uint32), cfg["layers"])
        tags = np.stack([np.full(n, seed & 0xFFFF, np.uint32), layer, block], axis=-1)
        kvx.fill_pages(pool, d_src, torch.from_numpy(tags.view(np.int32)).to(dev), n, seed, layout,
                       kvx.FILL_VALUES)
    return layout, pool, d_src, d_dst, src_ids, dst_ids


LAUNCHES = {"timed": 0}  # libkvx kernel launches inside the last time_events timed loop


def time_events(torch, fn, steps, warmup, marks=1):
    """Runs fn(i, ev_list) steps times after warmup; fn records marks+1 events."""
    from paper_2412_16434_b200 import kvx
    for i in range(warmup):
        fn(i, None)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(marks + 1)] for _ in range(steps)]
    n0 = kvx.launch_count()
    for i in range(steps):
        fn(i, evs[i])
    LAUNCHES["timed"] = kvx.launch_count() - n0
    torch.cuda.synchronize()
    total = evs[0][0].elapsed_time(evs[-1][-1])
    parts = [[e[j].elapsed_time(e[j + 1]) for e in evs] for j in range(marks)]
    return total, parts


def bench_single(args, torch, np, kvx, dev, hbm_peak, peak_kind):
    cfg = CFG_8B
    blocks, n = session_pages(cfg)
    layout, pool, d_src, d_dst, src_ids, dst_ids = make_session(torch, kvx, np, cfg, 1, dev)
    pb = layout.page_bytes()
    session_bytes = n * pb
    buf = torch.empty(session_bytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    mode = {"auto": kvx.COPY_AUTO, "sm": kvx.COPY_SM, "tma": kvx.COPY_TMA}[args.copy_mode]

    def step(i, ev, m=mode):
        if ev:
            ev[0].record(stream)
        kvx.pack(pool, d_src, n, buf, m, stream)
        if ev:
            ev[1].record(stream)
        kvx.unpack(pool, d_dst, n, buf, m, stream)
        if ev:
            ev[2].record(stream)

    with ClockSampler(dev.index) as clocks:
        total_ms, (pack_ms, unpack_ms) = time_events(torch, step, args.steps, args.warmup, marks=2)
    launches = LAUNCHES["timed"]  # counted by libkvx (kvx_launch_count), not inferred
    # correctness of what was timed: the last unpack landed every page
    probe = torch.randint(0, n, (64,), device=dev)
    pv = pool.as_tensor()
    assert torch.equal(pv[d_src[probe].long()], pv[d_dst[probe].long()]), "migrated pages differ"

    ms_per_step = total_ms / args.steps
    value = session_bytes / (ms_per_step * 1e-3) / GB
    pack_avg, unpack_avg = statistics.mean(pack_ms), statistics.mean(unpack_ms)
    dom_name, dom_ms = ("kvx_pack", pack_avg) if pack_avg >= unpack_avg else ("kvx_unpack", unpack_avg)
    achieved = 2 * session_bytes / (dom_ms * 1e-3) / GB  # read + write per launch
    extra = {
        "pack_ms": pack_avg, "unpack_ms": unpack_avg,
        "pack_hbm_gbs": 2 * session_bytes / (pack_avg * 1e-3) / GB,
        "unpack_hbm_gbs": 2 * session_bytes / (unpack_avg * 1e-3) / GB,
    }

    # Variants (not the headline): other copy mode, fused page->page K3.
    other = kvx.COPY_SM if mode in (kvx.COPY_AUTO, kvx.COPY_TMA) else kvx.COPY_TMA  # AUTO = TMA for HBM<->HBM
    _, (p2, u2) = time_events(torch, lambda i, ev: step(i, ev, other), max(5, args.steps // 2), 2, marks=2)
    extra["alt_mode"] = "tma" if other == kvx.COPY_TMA else "sm"
    extra["alt_pack_hbm_gbs"] = 2 * session_bytes / (statistics.mean(p2) * 1e-3) / GB
    extra["alt_unpack_hbm_gbs"] = 2 * session_bytes / (statistics.mean(u2) * 1e-3) / GB

    def fused(i, ev):
        if ev:
            ev[0].record(stream)
        kvx.copy_pages(pool, d_src, pool, d_dst, n, mode, stream)
        if ev:
            ev[1].record(stream)

    _, (fz,) = time_events(torch, fused, max(5, args.steps // 2), 2)
    extra["fused_copy_ms"] = statistics.mean(fz)
    extra["fused_copy_hbm_gbs"] = 2 * session_bytes / (statistics.mean(fz) * 1e-3) / GB
    extra["fused_copy_migrate_gbs"] = session_bytes / (statistics.mean(fz) * 1e-3) / GB
    del buf

    attention = None if args.skip_attention else bench_attention(args, torch, np, kvx, dev, hbm_peak)
    e2e_kvx = None if args.skip_e2e else bench_e2e(args, torch, np, kvx, dev, cfg, layout, pool, d_dst)
    overlap = None if args.skip_overlap else bench_overlap(args, torch, np, kvx, dev, hbm_peak)
    store_cycle = None if args.skip_e2e else bench_store_cycle(args, torch, np, kvx, dev)
    # e2e (the headline against the reference arm): the store's own API — the
    # reference-facing KvStore surface through the kvs C ABI — relocating
    # sessions between the pinned HOST tier and HBM pages: Symphony's swap
    # (offload A, load advised B; 1 GiB each way, host<->device copies and
    # the store's bookkeeping inside the timed region, bytes verified).
    # e2e (the headline against the reference arm): the same operation the
    # reference arm times — a session's migration through the store API
    # (mark_migrating_out -> import_migration -> apply every NetArrive ->
    # release), with real pages moved by K3, block tables uploaded and a
    # probe page read back inside the timed region.
    e2e = None if args.skip_e2e else bench_store_migration(args, torch, np, kvx, dev)
    if store_cycle is not None:
        sw = store_cycle["swap"]
        extra["e2e_store_swap"] = {
            "value": sw["value"], "unit": UNIT, "h2d_bytes_per_step": session_bytes,
            "d2h_bytes_per_step": session_bytes, "ms_per_step": sw["ms_per_swap"], "steps": sw["swaps"],
            "path": "kvs_offload_session(A: HBM pages -> pinned HOST) + kvs_plan_layerwise_load(B: pinned HOST "
                    "-> HBM pages), NodePayload free-running, both PCIe directions"}
    if e2e_kvx is not None:
        extra["e2e_kvx_roundtrip"] = e2e_kvx
    disk = None if args.skip_e2e else bench_disk(args, torch, np, kvx, cfg)
    return dict(value=value, ms_per_step=ms_per_step, extra=extra, clocks=clocks.summary(),
                roofline={"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                          "frac": achieved / hbm_peak, "traffic": ncu_traffic(dom_name), "kernel": dom_name,
                          "algorithmic_bytes_per_launch": 2 * session_bytes, "peak_kind": peak_kind,
                          "frac_of_nominal_8tbs": achieved / 8000.0},
                attention=attention, e2e=e2e, overlap=overlap, store_cycle=store_cycle, disk_tier=disk,
                gpu_launches=launches,
                session_bytes=session_bytes)


def graph_time_ms(torch, launch, reps, replays, warmup=2):
    """Per-launch device time of `launch(i)` captured `reps` times into one
    CUDA graph (decode loops replay graphs; this keeps host launch overhead
    out of a microsecond-scale kernel's number), replayed `replays` times."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(warmup):
            launch(i)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            launch(i)
    g.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(replays):
        g.replay()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / (replays * reps)


def bench_attention(args, torch, np, kvx, dev, hbm_peak):
    """K4 over one layer of Llama-3.1-8B KV at ctx 8192 (GQA 32/8) at batch
    1/8/64, and of Llama-3.1-70B KV at ctx 32768 (GQA 64/8) at batch 1/4;
    launches replayed from a CUDA graph, rotating request sets so
    consecutive launches read >= 256 MiB (> L2)."""
    cfg = CFG_8B
    blocks = cfg["ctx"] // cfg["block_tokens"]
    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    pb = layout.page_bytes()
    max_b = 64
    pages = max_b * blocks
    rng = np.random.default_rng(3)
    pool = kvx.Pool(pages, pb, device=dev.index)
    ids = torch.arange(pages, dtype=torch.int32, device=dev)
    tags = torch.stack([torch.zeros_like(ids), torch.zeros_like(ids), ids], -1).contiguous()
    kvx.fill_pages(pool, ids, tags, pages, 5, layout, kvx.FILL_VALUES)
    perm = torch.from_numpy(rng.permutation(pages).astype(np.int32)).to(dev)
    res = {}
    for batch in (1, 8, 64):
        sets = max(1, min(pages // (batch * blocks), -(-256 // (batch * 32))))
        tables = [perm[s * batch * blocks:(s + 1) * batch * blocks].view(batch, blocks).contiguous()
                  for s in range(sets)]
        ctx = torch.full((batch,), cfg["ctx"], dtype=torch.int32, device=dev)
        q = (torch.randn(batch, 32, 128, device=dev) * 0.5).to(torch.bfloat16)
        out = torch.empty(batch, 32, 128, dtype=torch.float32, device=dev)
        kv_bytes = batch * cfg["ctx"] * 2 * cfg["kv_heads"] * cfg["head_dim"] * 2
        reps = max(sets, 16 if batch < 64 else 4)

        def timed(splits, merge=kvx.MERGE_AUTO):
            att = kvx.Attention(layout, 32, blocks, num_splits=splits, split_merge=merge, flags=DECODE_FLAGS(kvx))
            ws = torch.zeros(max(att.workspace_bytes(batch, cfg["ctx"]), 1), dtype=torch.uint8, device=dev)
            return graph_time_ms(torch, lambda i: att(pool, tables[i % sets], ctx, q, out, batch, cfg["ctx"], ws),
                                 reps, max(3, min(args.steps, 20)))

        t = timed(0)
        gbs = kv_bytes / (t * 1e-3) / GB
        res[f"batch{batch}"] = {"ms_per_layer": t, "hbm_gbs": gbs, "frac": gbs / hbm_peak,
                                "kv_bytes": kv_bytes, "rotating_sets": sets, "timing": "cuda-graph replay"}
        if args.attn_sweep:  # diagnostic: fixed split-K factors
            res[f"batch{batch}"]["split_sweep_gbs"] = {
                s: round(kv_bytes / (timed(s, kvx.MERGE_GLOBAL) * 1e-3) / GB, 1)
                for s in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32)}
            res[f"batch{batch}"]["cluster_sweep_gbs"] = {
                s: round(kv_bytes / (timed(s, kvx.MERGE_CLUSTER) * 1e-3) / GB, 1)
                for s in (2, 3, 4, 6, 8, 9, 12, 16) if batch * cfg["kv_heads"] * s <= 148}
    # One decode step of one layer as the engine runs it (append this token's
    # K/V, then attend): kvx_append_kv + kvx_decode_attention (two launches)
    # vs kvx_decode_attention_append (append fused into the attention launch).
    for batch in (1, 8):
        sets = max(1, min(pages // (batch * blocks), -(-256 // (batch * 32))))
        tables = [perm[s * batch * blocks:(s + 1) * batch * blocks].view(batch, blocks).contiguous()
                  for s in range(sets)]
        ctx = torch.full((batch,), cfg["ctx"], dtype=torch.int32, device=dev)
        q = (torch.randn(batch, 32, 128, device=dev) * 0.5).to(torch.bfloat16)
        nk = (torch.randn(batch, cfg["kv_heads"], 128, device=dev) * 0.5).to(torch.bfloat16)
        nv = (torch.randn(batch, cfg["kv_heads"], 128, device=dev) * 0.5).to(torch.bfloat16)
        out = torch.empty(batch, 32, 128, dtype=torch.float32, device=dev)
        slots = torch.full((batch,), (cfg["ctx"] - 1) % cfg["block_tokens"], dtype=torch.int32, device=dev)
        last = [t[:, (cfg["ctx"] - 1) // cfg["block_tokens"]].contiguous() for t in tables]
        att = kvx.Attention(layout, 32, blocks, flags=DECODE_FLAGS(kvx))
        ws = torch.zeros(max(att.workspace_bytes(batch, cfg["ctx"]), 1), dtype=torch.uint8, device=dev)
        reps, replays = max(sets, 16), max(3, min(args.steps, 20))

        def two(i):
            kvx.append_kv(pool, layout, last[i % sets], slots, nk, nv, batch)
            att(pool, tables[i % sets], ctx, q, out, batch, cfg["ctx"], ws)

        t_two = graph_time_ms(torch, two, reps, replays)
        t_fused = graph_time_ms(torch, lambda i: att(pool, tables[i % sets], ctx, q, out, batch, cfg["ctx"], ws,
                                                     new_k=nk, new_v=nv), reps, replays)
        res[f"decode_step_batch{batch}"] = {"append_then_attend_ms": t_two, "fused_ms": t_fused,
                                            "speedup": t_two / t_fused, "timing": "cuda-graph replay, per layer"}
    # Config 3's decode shape: Llama-3.1-70B (64 q heads over 8 kv heads, GQA 8) at ctx 32768.
    c70 = CFG_70B
    blocks70 = c70["ctx"] // c70["block_tokens"]
    for batch in (1, 4):
        sets = max(1, min(pages // (batch * blocks70), -(-256 // (batch * 128))))
        tables = [perm[s * batch * blocks70:(s + 1) * batch * blocks70].view(batch, blocks70).contiguous()
                  for s in range(sets)]
        ctx = torch.full((batch,), c70["ctx"], dtype=torch.int32, device=dev)
        q = (torch.randn(batch, 64, 128, device=dev) * 0.5).to(torch.bfloat16)
        out = torch.empty(batch, 64, 128, dtype=torch.float32, device=dev)
        kv_bytes = batch * c70["ctx"] * 2 * c70["kv_heads"] * c70["head_dim"] * 2
        att = kvx.Attention(layout, 64, blocks70, flags=DECODE_FLAGS(kvx))
        ws = torch.zeros(max(att.workspace_bytes(batch, c70["ctx"]), 1), dtype=torch.uint8, device=dev)
        t = graph_time_ms(torch, lambda i: att(pool, tables[i % sets], ctx, q, out, batch, c70["ctx"], ws),
                          max(sets, 8), max(3, min(args.steps, 20)))
        gbs = kv_bytes / (t * 1e-3) / GB
        res[f"llama70b_ctx32k_batch{batch}"] = {"ms_per_layer": t, "hbm_gbs": gbs, "frac": gbs / hbm_peak,
                                                "kv_bytes": kv_bytes, "rotating_sets": sets,
                                                "timing": "cuda-graph replay"}
    return res


def bench_overlap(args, torch, np, kvx, dev, hbm_peak):
    """Migration overlapped with decode, on one GPU (free-running streams).

    decode : one decode step of Llama-3.1-8B KV at batch 16 x ctx 8192 — 32
             layers of K4 on the main stream (17 GB of KV read per step)
    migrate: one 8B@8K session (1 GiB) moved layer by layer with K3 on a side
             stream (SM mover, or copy engines), one event per layer
    Both are CUDA graphs; the concurrent case is one graph that forks the side
    stream. Reported: decode slowdown and the hidden fraction of the
    migration. Then the physical pipeline gate: a batch-1 decode of the
    migrating session whose layer l waits on layer l's arrival event,
    against pipeline_gate()'s prediction from the measured arrivals
    (reference kvstore.cpp:46-59)."""
    from paper_2412_16434_b200 import kvstore as K
    cfg = CFG_8B
    L, blocks = cfg["layers"], cfg["ctx"] // cfg["block_tokens"]
    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    pb = layout.page_bytes()
    B = args.bg_batch  # decode batch (16 default; 64 = config 5's decode batches)
    dec_pages = B * L * blocks
    dpool = kvx.Pool(dec_pages, pb, device=dev.index)
    ids = torch.arange(dec_pages, dtype=torch.int32, device=dev)
    kvx.fill_pages(dpool, ids, torch.stack([ids * 0, ids * 0, ids], -1).contiguous(), dec_pages, 11, layout,
                   kvx.FILL_VALUES)
    perm = torch.randperm(dec_pages, device=dev, dtype=torch.int64).to(torch.int32)
    tables = [perm[l * B * blocks:(l + 1) * B * blocks].view(B, blocks).contiguous() for l in range(L)]
    ctx = torch.full((B,), cfg["ctx"], dtype=torch.int32, device=dev)
    q = (torch.randn(B, 32, 128, device=dev) * 0.5).to(torch.bfloat16)
    out = torch.empty(B, 32, 128, dtype=torch.float32, device=dev)
    att = kvx.Attention(layout, 32, blocks, flags=DECODE_FLAGS(kvx))
    ws = torch.zeros(max(att.workspace_bytes(B, cfg["ctx"]), 1), dtype=torch.uint8, device=dev)

    n = L * blocks
    spool = kvx.Pool(2 * n, pb, device=dev.index)
    sp = torch.randperm(2 * n, device=dev, dtype=torch.int64).to(torch.int32)
    src, dst = sp[:n].contiguous(), sp[n:].contiguous()
    kvx.fill_pages(spool, src, torch.stack([src * 0 + 3, src // blocks, src % blocks], -1).contiguous(), n, 3,
                   layout, kvx.FILL_VALUES)
    h_src = src.cpu().numpy().view(np.uint32)
    h_dst = dst.cpu().numpy().view(np.uint32)
    q1 = q[:1].contiguous()
    out1 = torch.empty(1, 32, 128, dtype=torch.float32, device=dev)
    ctx1 = ctx[:1].contiguous()
    att1 = kvx.Attention(layout, 32, blocks, flags=DECODE_FLAGS(kvx))
    ws1 = torch.zeros(max(att1.workspace_bytes(1, cfg["ctx"]), 1), dtype=torch.uint8, device=dev)
    mig_tables = [dst[l * blocks:(l + 1) * blocks].view(1, blocks).contiguous() for l in range(L)]
    torch.cuda.synchronize()

    side = torch.cuda.Stream(dev)

    def decode(st):
        for l in range(L):
            att(dpool, tables[l], ctx, q, out, B, cfg["ctx"], ws, st.cuda_stream)

    def migrate(st, mode, events=None):
        for l in range(L):
            sl = slice(l * blocks, (l + 1) * blocks)
            if mode == kvx.COPY_CE:
                kvx.copy_pages(spool, h_src[sl], spool, h_dst[sl], blocks, mode, st.cuda_stream)
            else:
                kvx.copy_pages(spool, src[sl], spool, dst[sl], blocks, mode, st.cuda_stream)
            if events is not None:
                events[l].record(st)

    def capture(body):
        cap = torch.cuda.Stream(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            body(cap)
        return g

    def time_graph(g, reps=10):
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(reps):
            g.replay()
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / reps

    def fork(cap, fn):
        side.wait_stream(cap)
        with torch.cuda.stream(side):
            fn(side)
        cap.wait_stream(side)

    res = {"decode": f"batch {B} x ctx {cfg['ctx']} x {L} layers (K4)", "migration": "1 GiB session, 32 layer moves"}
    t_dec = time_graph(capture(lambda c: decode(c)))
    res["decode_alone_ms"] = t_dec
    for name, mode in (("sm", kvx.COPY_AUTO), ("ce", kvx.COPY_CE)):
        t_mig = time_graph(capture(lambda c: migrate(c, mode)))
        t_both = time_graph(capture(lambda c: (fork(c, lambda st: migrate(st, mode)), decode(c))))
        res[name] = {"migrate_alone_ms": t_mig, "concurrent_ms": t_both,
                     "decode_slowdown": t_both / t_dec - 1.0,
                     "hidden_fraction": max(0.0, min(1.0, (t_dec + t_mig - t_both) / t_mig)),
                     "migrate_gbs_alone": n * pb / (t_mig * 1e-3) / GB,
                     "note": "decode and a full-speed local migration are both HBM-bound on one GPU, so the "
                             "migration's bytes are shared rather than hidden; `background` measures the cost "
                             "per GiB against the HBM floor"}

    def migrate_capped(st, mode, cap):
        for l in range(L):
            sl = slice(l * blocks, (l + 1) * blocks)
            kvx.copy_pages(spool, src[sl], spool, dst[sl], blocks, mode, st.cuda_stream, max_ctas=cap)

    res["background"] = background_migration(torch, kvx, decode, migrate_capped, side, dev, n * pb, t_dec,
                                             hbm_peak, sweep=args.bg_sweep)

    # Physical pipeline gate: per-layer arrival events gate a batch-1 decode of
    # the migrating session; compare with the reference recurrence.
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(L)]
    t0 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(side)
    migrate(side, kvx.COPY_AUTO, ev)
    torch.cuda.synchronize()
    ready_us = [t0.elapsed_time(e) * 1e3 for e in ev]
    t_layer = time_graph(capture(lambda c: [att1(spool, mig_tables[l], ctx1, q1, out1, 1, cfg["ctx"], ws1,
                                                 c.cuda_stream) for l in range(L)])) / L

    def gated(c):
        evs = [torch.cuda.Event() for _ in range(L)]
        side.wait_stream(c)
        with torch.cuda.stream(side):
            migrate(side, kvx.COPY_AUTO, evs)
        for l in range(L):
            c.wait_event(evs[l])
            att1(spool, mig_tables[l], ctx1, q1, out1, 1, cfg["ctx"], ws1, c.cuda_stream)
        c.wait_stream(side)

    t_gated = time_graph(capture(gated))
    ns = [int(r * 1e3) for r in ready_us]
    first_end, gate_start, stall = K.pipeline_gate(ns, 0, int(L * t_layer * 1e6))
    res["pipeline_gate"] = {"layer_arrival_us_first_last": [ready_us[0], ready_us[-1]],
                            "layer_decode_us": t_layer * 1e3, "measured_first_step_end_us": t_gated * 1e3,
                            "predicted_first_step_end_us": first_end / 1e3, "predicted_stall_us": stall / 1e3,
                            "unpipelined_us": ready_us[-1] + L * t_layer * 1e3}
    return res


def background_migration(torch, kvx, decode, migrate, side, dev, session_bytes, t_step, hbm_peak, sweep=False):
    """Serving with a session migrating underneath, on one GPU.

    Decode runs `steps` back-to-back steps on a high-priority stream while one
    session migrates on a low-priority side stream with the mover's grid
    capped to `cap` CTAs (kvx_copy_pages_capped). In an N-GPU ring each GPU
    reads the session it sends and writes the one it receives, so its HBM sees
    the same read + write bytes as this local copy: this measures the HBM side
    of "migration hidden behind decode" (NVLink itself needs two GPUs).
    Reported per variant: migration GB/s while decode runs (vs the 770 GB/s
    NVLink peer-copy peak), the decode time added over `steps` steps, and the
    floor — the HBM time the migration's read + write bytes need at the
    measured copy peak (what an ideal share of HBM would add)."""
    steps = 4
    floor = 2 * session_bytes / (hbm_peak * GB) * 1e3
    out = {"decode_steps": steps, "decode_step_ms_alone": t_step, "hbm_peak_gbs": hbm_peak,
           "hbm_floor_extra_ms": floor, "variants": [],
           "note": "same-GPU HBM copy: hbm_frac is the migration's read + write bytes over the measured HBM copy "
                   "peak while decode runs; no NVLink is involved on one GPU"}
    hi = torch.cuda.Stream(dev, priority=-5)   # clamped to the device's highest priority
    lo = torch.cuda.Stream(dev, priority=0)
    if sweep:
        variants = [(m, cap, geo, prio) for m in ("tma", "sm") for cap in (8, 16, 24, 32, 48, 74, 0)
                    for geo in ((None,) if m == "sm" else (None, (8192, 3), (16384, 2)))
                    for prio in (False, True)]
    else:
        # the measured-best rows of the sweep (profiles/r01_background_sweep.json)
        variants = [("tma", 0, None, False), ("tma", 48, None, False), ("sm", 0, None, False),
                    ("sm", 74, None, False)]
    modes = {"tma": kvx.COPY_TMA, "sm": kvx.COPY_SM}
    saved = {k: os.environ.get(k) for k in ("KVX_BULK_CHUNK", "KVX_BULK_STAGES")}

    def run(dec_st, mig_st, mode, cap):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        ev[0].record(dec_st)
        mig_st.wait_event(ev[0])
        if mode is not None:
            migrate(mig_st, mode, cap)
        ev[1].record(mig_st)
        for _ in range(steps):
            decode(dec_st)
        ev[2].record(dec_st)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]), ev[0].elapsed_time(ev[2])

    try:
        for prio in (False, True):  # decode alone on each stream kind (same work, reference point)
            dec_st = hi if prio else torch.cuda.current_stream(dev)
            out["decode_alone_ms_" + ("hi" if prio else "default")] = statistics.median(
                run(dec_st, lo, None, 0)[1] for _ in range(3))
        for mname, cap, geo, prio in variants:
            for k in saved:
                os.environ.pop(k, None)
            if geo:
                os.environ["KVX_BULK_CHUNK"], os.environ["KVX_BULK_STAGES"] = str(geo[0]), str(geo[1])
            dec_st = hi if prio else torch.cuda.current_stream(dev)
            mig_st = lo if prio else side
            base = out["decode_alone_ms_" + ("hi" if prio else "default")]
            rows = [run(dec_st, mig_st, modes[mname], cap) for _ in range(3)]
            t_mig = statistics.median(r[0] for r in rows)
            t_all = statistics.median(r[1] for r in rows)
            extra = max(0.0, t_all - base)
            out["variants"].append({
                "mover": mname, "max_ctas": cap or "all", "stage": f"{geo[0] // 1024}KiBx{geo[1]}" if geo else "default",
                "priority_streams": prio, "migrate_ms": t_mig, "migrate_gbs": session_bytes / (t_mig * 1e-3) / GB,
                "hbm_frac": 2 * session_bytes / (t_mig * 1e-3) / GB / hbm_peak, "decode_ms": t_all,
                "decode_extra_ms": extra, "extra_over_floor": extra / floor})
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return out


def bench_disk(args, torch, np, kvx, cfg):
    """DISK tier as a file (kvx_pool_create_file): one 8B@8K session (1 GiB)
    written from a pinned HOST pool to the file at a random page placement
    (DiskWrite, kvstore.cpp:881-900) and read back into a second HOST pool
    (LoadDiskHost, :862-866) with kvx_copy_pages(COPY_CE): preads / pwrites
    in stream order, O_DIRECT where the filesystem allows. Device-timed with
    CUDA events around the host callbacks; bytes verified."""
    import shutil
    import tempfile
    blocks, n = session_pages(cfg)
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    host = kvx.Pool(n, pb, host=True)
    back = kvx.Pool(n, pb, host=True)
    host.as_tensor().view(torch.int64).random_()
    d = tempfile.mkdtemp(prefix="kvx_disk_", dir=os.environ.get("KVX_DISK_DIR", "/tmp"))
    try:
        disk = kvx.Pool.file(os.path.join(d, "disk.pages"), n, pb)
        ids = np.arange(n, dtype=np.uint32)
        place = np.random.default_rng(11).permutation(n).astype(np.uint32)
        st = torch.cuda.Stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(st)
        kvx.copy_pages(host, ids, disk, place, n, kvx.COPY_CE, stream=st)
        ev[1].record(st)
        kvx.copy_pages(disk, place, back, ids, n, kvx.COPY_CE, stream=st)
        ev[2].record(st)
        st.synchronize()
        probe = np.random.default_rng(12).integers(0, n, 256)
        assert torch.equal(back.as_tensor()[probe], host.as_tensor()[probe]), "disk round trip differs"
        w_ms, r_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        res = {"bytes": n * pb, "write_gbs": n * pb / (w_ms * 1e-3) / GB, "read_gbs": n * pb / (r_ms * 1e-3) / GB,
               "o_direct": disk.direct_io, "pages": n, "page_bytes": pb, "placement": "random page order",
               "path": "pinned HOST pool <-> file pool, kvx_copy_pages(COPY_CE), 8 I/O threads"}
        disk.close()
        return res
    finally:
        shutil.rmtree(d, ignore_errors=True)


def bench_store_cycle(args, torch, np, kvx, dev):
    """The store-driven tier cycle of one 8B @8K session through the kvs C ABI
    (KvStore + NodePayload, free-running): offload_session (32 per-layer
    SwapOut moves DEVICE -> pinned HOST, copy engines) then
    plan_layerwise_load (32 LoadH2D moves back to fresh DEVICE pages), with
    the cost model calibrated to the measured PCIe rate. Every move is issued
    when the store schedules it and completed when the transfer is applied in
    (complete_at, id) order; the host only waits if the GPU is behind."""
    from paper_2412_16434_b200 import kvstore as K
    cfg = CFG_8B
    blocks, n = session_pages(cfg)
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    gpu = K.GpuProfile(kv_bytes_per_token=cfg["layers"] * pb // cfg["block_tokens"], num_layers=cfg["layers"],
                       hbm_capacity=100 * n * pb)
    links = K.LinkProfile(pcie_bandwidth=55e9)
    st = K.KvStore(gpu=gpu, links=links, opts=K.Options(write_behind=False, host_capacity=4 * n * pb))
    node = K.NodePayload(K.PayloadCluster(), 0, K.PayloadOptions(
        device=dev.index, num_kv_heads=cfg["kv_heads"], head_dim=cfg["head_dim"], dtype=kvx.BF16,
        device_pages=2 * n, host_pages=n, landing_pages=1, disk_pages=1, seed=9, free_running=True))
    node.attach(st)
    steps = max(3, min(args.steps, 8))
    for i in range(steps + 1):  # a fresh session per cycle: its only copy starts on DEVICE
        st.register_session(i, f"s{i}")
    st.finalize_sessions()

    def pump(sched):
        for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
            st.apply_transfer(tid, at)

    now = 1_000_000
    times = []
    for i in range(steps + 1):
        _, sched = st.append_blocks(i, cfg["ctx"], now)  # untimed: creation fills the pages
        pump(sched)
        node.synchronize()
        t0 = time.perf_counter()
        pump(st.offload_session(i, now + 1))  # 1 GiB DEVICE -> HOST
        plan, sched = st.plan_layerwise_load(i, now + 2, 1000, K.DEMAND)  # 1 GiB HOST -> DEVICE
        pump(sched)
        node.synchronize()
        if i:  # first cycle is warm-up
            times.append(time.perf_counter() - t0)
        assert st.fully_device_resident(i)
        st.release_session(i, now + 3)
        now += 10_000_000_000
    t = statistics.mean(times)
    st_ = node.stats()
    res = {"value": 2 * n * pb / t / GB, "unit": "GB/s (D2H + H2D session bytes)", "ms_per_cycle": 1e3 * t,
           "cycles": steps, "apply_wait_ms_total": st_["apply_wait_ns"] / 1e6,
           "transfers_issued_at_schedule_time": st_["transfers_posted"],
           "path": "kvs_offload_session + kvs_plan_layerwise_load, NodePayload free-running (copy engines)"}
    res["swap"] = bench_store_swap(args, K, kvx, cfg, n, pb, dev)
    return res


def bench_store_migration(args, torch, np, kvx, dev):
    """The e2e headline, the same operation as the reference arm: a session's
    migration through the store API (the reference's
    Simulation::start_migration, simcore.cpp:132-141): kvs_mark_migrating_out
    on the source node, kvs_import_migration on the receiver (one NetArrive
    per layer, kvstore.cpp:744-789), every NetArrive applied in (complete_at,
    id) order (kvstore.cpp:914-923), kvs_release_session on the source
    (kvstore.cpp:710-736). With the payload free-running, each layer's arrival
    is a K3 push of the source's HBM pages into the receiver's landing pool,
    issued when import_migration schedules it and completed at apply. Two
    nodes share this GPU (on a multi-GPU box the push crosses NVLink). Inside
    the host-timed region per step: the store bookkeeping of both nodes, the
    block-table uploads from host memory (the page-id lists of every layer,
    H2D), the GPU moves, and a probe page read back to host memory (D2H);
    the probe is verified against the block's content."""
    from paper_2412_16434_b200 import kvstore as K
    cfg = CFG_8B
    blocks, n = session_pages(cfg)
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    gpu = K.GpuProfile(kv_bytes_per_token=cfg["layers"] * pb // cfg["block_tokens"], num_layers=cfg["layers"],
                       hbm_capacity=100 * n * pb)
    links = K.LinkProfile(network_bandwidth=770e9)
    cluster = K.PayloadCluster()
    stores, nodes = [], []
    for node_id in range(2):
        st = K.KvStore(gpu=gpu, links=links, opts=K.Options(node_id=node_id, write_behind=False,
                                                           host_capacity=4 * n * pb))
        nd = K.NodePayload(cluster, node_id, K.PayloadOptions(
            device=dev.index, num_kv_heads=cfg["kv_heads"], head_dim=cfg["head_dim"], dtype=kvx.BF16,
            device_pages=2 * n if node_id == 0 else 1, host_pages=1, landing_pages=2 * n if node_id else 1,
            disk_pages=1, seed=17, free_running=True))
        nd.attach(st)
        stores.append(st)
        nodes.append(nd)
    src, dst = stores
    steps = max(3, min(args.steps, 10))
    for st in stores:
        for i in range(steps + 1):
            st.register_session(i, f"m{i}")
        st.finalize_sessions()

    def pump(store, sched):
        for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
            store.apply_transfer(tid, at)

    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    ref = kvx.Pool(1, pb, device=dev.index)
    now, times, verified = 1_000_000, [], 0
    rng = np.random.default_rng(3)
    for i in range(steps + 1):
        _, sched = src.append_blocks(i, cfg["ctx"], now)  # untimed: the session to migrate
        pump(src, sched)
        nodes[0].synchronize()
        layer, block = int(rng.integers(cfg["layers"])), int(rng.integers(blocks))
        t0 = time.perf_counter()
        src.mark_migrating_out(i)
        pump(dst, dst.import_migration(i, cfg["ctx"], now + 1))
        src.release_session(i, now + 2)
        probe = nodes[1].read_block(i, layer, block, K.HOST, pb)  # syncs the payload, D2H of one page
        dt = time.perf_counter() - t0
        if i:
            times.append(dt)
        kvx.fill_pages(ref, torch.zeros(1, dtype=torch.int32, device=dev),
                       torch.tensor([[i, layer, block]], dtype=torch.int32, device=dev), 1, 17, layout,
                       kvx.FILL_VALUES)
        torch.cuda.synchronize()
        assert probe is not None and np.array_equal(probe, ref.as_tensor().cpu().numpy()[0]), "migrated page differs"
        verified += 1
        dst.release_session(i, now + 3)  # untimed: frees the landing pages for the next step
        now += 10_000_000_000
    t = statistics.mean(times)
    ids_bytes = 2 * n * 4  # source + destination page ids of every layer, uploaded per step
    host = nodes[1].host_ns()
    return {"value": n * pb / t / GB, "unit": UNIT, "h2d_bytes_per_step": ids_bytes, "d2h_bytes_per_step": pb,
            "ms_per_step": 1e3 * t, "steps": len(times), "verified_probe_pages": verified,
            "copies_declared": True,
            "timing": "host wall clock around the store calls, the payload's GPU moves and the probe read",
            "path": "kvs_mark_migrating_out(src) -> kvs_import_migration(dst) -> kvs_apply_transfer x32 "
                    "(NetArrive: K3 push into dst's landing pool) -> kvs_release_session(src) -> probe page D2H",
            "receiver_host_us_per_layer": {k: round(v / 1e3 / cfg["layers"] / (steps + 1), 2)
                                           for k, v in host.items() if k in ("posted", "retired", "issue")}}


def bench_store_swap(args, K, kvx, cfg, n, pb, dev):
    """Symphony's tier swap on one node: while session A is offloaded (SwapOut,
    DEVICE -> HOST) session B, advised to arrive, is loaded back (LoadH2D,
    HOST -> DEVICE). Both are posted together and applied in the store's
    (complete_at, id) order; the payload runs them on its OUT and IN lanes, so
    the two PCIe directions overlap. Value: session bytes moved per second,
    both directions counted."""
    gpu = K.GpuProfile(kv_bytes_per_token=cfg["layers"] * pb // cfg["block_tokens"], num_layers=cfg["layers"],
                       hbm_capacity=100 * n * pb)
    st = K.KvStore(gpu=gpu, links=K.LinkProfile(pcie_bandwidth=55e9),
                   opts=K.Options(write_behind=False, host_capacity=8 * n * pb))
    node = K.NodePayload(K.PayloadCluster(), 0, K.PayloadOptions(
        device=dev.index, num_kv_heads=cfg["kv_heads"], head_dim=cfg["head_dim"], dtype=kvx.BF16,
        device_pages=3 * n, host_pages=3 * n, landing_pages=1, disk_pages=1, seed=13, free_running=True))
    node.attach(st)
    cycles = max(3, min(args.steps, 8))
    for i in range(cycles + 2):
        st.register_session(i, f"w{i}")
    st.finalize_sessions()

    def pump(sched):
        for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
            st.apply_transfer(tid, at)

    def verify_swapped_in(b_sess):
        node.synchronize()
        return _verify_swapped_in(K, kvx, node, cfg, n, pb, dev, b_sess)

    verified = 0
    now = 1_000_000
    _, sched = st.append_blocks(0, cfg["ctx"], now)  # session 0 starts offloaded
    pump(sched)
    pump(st.offload_session(0, now + 1))
    node.synchronize()
    times = []
    for i in range(1, cycles + 2):
        now += 10_000_000_000
        _, sched = st.append_blocks(i, cfg["ctx"], now)  # A = i on DEVICE (untimed fill)
        pump(sched)
        node.synchronize()
        t0 = time.perf_counter()
        out = st.offload_session(i, now + 1)  # A: DEVICE -> HOST
        _, load = st.plan_layerwise_load(i - 1, now + 1, 1000, K.DEMAND)  # B = i - 1: HOST -> DEVICE
        pump(out + load)
        node.synchronize()
        if i > 1:
            times.append(time.perf_counter() - t0)
        assert st.fully_device_resident(i - 1)
        if i == cycles + 1:
            verified = verify_swapped_in(i - 1)
        st.release_session(i - 1, now + 2)
    t = statistics.mean(times)
    s = node.stats()
    return {"value": 2 * n * pb / t / GB, "unit": "GB/s (D2H + H2D session bytes, concurrent)",
            "ms_per_swap": 1e3 * t, "swaps": len(times), "cross_lane_waits": s["cross_lane_waits"],
            "verified_blocks": verified,
            "path": "kvs_offload_session(A) + kvs_plan_layerwise_load(B) posted together, IN/OUT lanes"}


def _verify_swapped_in(K, kvx, node, cfg, n, pb, dev, b_sess):
    """What a swap loaded is session B's content, bit for bit (creation filled
    each (session, layer, block) from seed 13 with the KVX_FILL_VALUES rule)."""
    import torch
    import numpy as np
    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    rng = np.random.default_rng(5)
    probe = [(int(l), int(b))
             for l, b in zip(rng.integers(0, cfg["layers"], 16), rng.integers(0, n // cfg["layers"], 16))]
    ref = kvx.Pool(len(probe), pb, device=dev.index)
    tags = torch.tensor([[b_sess, l, b] for l, b in probe], dtype=torch.int32, device=dev)
    kvx.fill_pages(ref, torch.arange(len(probe), dtype=torch.int32, device=dev), tags, len(probe), 13, layout,
                   kvx.FILL_VALUES)
    torch.cuda.synchronize()
    want = ref.as_tensor().cpu().numpy()
    for i, (l, b) in enumerate(probe):
        got = node.read_block(b_sess, l, b, K.DEVICE, pb)
        assert got is not None and np.array_equal(got, want[i]), f"swapped-in block ({l}, {b}) differs"
    return len(probe)


def bench_e2e(args, torch, np, kvx, dev, cfg, layout, pool, d_dst):
    """Through the C ABI with pinned HOST buffers: per layer H2D (HOST tier copy
    -> staging) + unpack (K2, LoadH2D landing) + pack (K1, offload gather) +
    D2H (-> HOST tier). Copy streams overlap the two PCIe directions."""
    blocks, n = session_pages(cfg)
    pb = layout.page_bytes()
    lb = blocks * pb
    L = cfg["layers"]
    h_in = torch.empty(L * lb, dtype=torch.uint8).pin_memory()
    h_in.view(torch.int64).random_()
    h_out = torch.empty_like(h_in).pin_memory()
    NB = 3  # staging slots per direction: H2D of layer g+2 overlaps compute of g+1 and D2H of g
    stage_in = [torch.empty(lb, dtype=torch.uint8, device=dev) for _ in range(NB)]
    stage_out = [torch.empty(lb, dtype=torch.uint8, device=dev) for _ in range(NB)]
    s_in, s_c, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    done_c, done_out = {}, {}  # global layer index -> event (slot reuse across step boundaries)

    def step(k):
        """Step k moves every layer in and out; layers of consecutive steps
        stream back to back (a slot waits only for the layer that last used
        it), as a serving node streams sessions through its HOST tier."""
        for l in range(L):
            g = k * L + l
            slot = g % NB
            with torch.cuda.stream(s_in):
                if g - NB in done_c:
                    s_in.wait_event(done_c.pop(g - NB))
                stage_in[slot].copy_(h_in[l * lb:(l + 1) * lb], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(s_in)
            s_c.wait_event(e_in)
            if g - NB in done_out:
                s_c.wait_event(done_out.pop(g - NB))
            ids = d_dst[l * blocks:(l + 1) * blocks]
            kvx.unpack(pool, ids, blocks, stage_in[slot], kvx.COPY_AUTO, s_c)
            kvx.pack(pool, ids, blocks, stage_out[slot], kvx.COPY_AUTO, s_c)
            e_c = torch.cuda.Event()
            e_c.record(s_c)
            done_c[g] = e_c
            with torch.cuda.stream(s_out):
                s_out.wait_event(e_c)
                h_out[l * lb:(l + 1) * lb].copy_(stage_out[slot], non_blocking=True)
                e_out = torch.cuda.Event()
                e_out.record(s_out)
                done_out[g] = e_out

    steps = max(3, min(args.steps, 10))
    warm = max(1, min(args.warmup, 3))
    for k in range(warm):
        step(k)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(main)
    s_in.wait_stream(main)
    for k in range(warm, warm + steps):
        step(k)
    main.wait_stream(s_out)
    t1.record(main)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    assert torch.equal(h_in, h_out), "end-to-end roundtrip differs"
    return {"value": (L * lb) / (ms * 1e-3) / GB, "unit": UNIT, "h2d_bytes_per_step": L * lb,
            "d2h_bytes_per_step": L * lb, "ms_per_step": ms, "steps": steps,
            "path": "pinned HOST -> H2D -> kvx_unpack -> kvx_pack -> D2H -> pinned HOST, per layer, 3 streams, "
                    "3 staging slots per direction, layers of consecutive steps streamed back to back"}


def bench_store_ring(args, torch, np, kvx, rank, world):
    """N>1 through the store API — the product path (config 3): the
    reference's Simulation::start_migration (simcore.cpp:132-141) per session,
    as the product runs it. One process drives a PayloadCluster of N nodes,
    node i on cuda:i (rank 0; the other ranks only hold the barrier), each
    node a KvStore + free-running NodePayload holding one Llama-3.1-70B @32K
    session. A step migrates every session one hop around the ring at once:
    mark_migrating_out on the holder, import_migration on the next node (80
    NetArrives, each a K3 push of the holder's pages into the receiver's
    landing pool, over NVLink when the nodes sit on different GPUs — peer
    access enabled by the payload on import), every NetArrive applied in
    (complete_at, id) order, release_session on the holder. The session
    travels on from the receiver's landing pool in the next step.

    Timing: CUDA events on each holder's PEER lane around the pushes; the
    step time is the max over the N devices (their migrations run
    concurrently); value = N x session bytes / that max. With --same-device
    every node sits on cuda:0 (test mode)."""
    import torch.distributed as dist
    from paper_2412_16434_b200 import kvstore as K
    cfg = dict(CFG_70B)
    if args.layers:
        cfg["layers"] = args.layers
    L = cfg["layers"]
    blocks, n = session_pages(cfg)
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    if rank != 0:
        dist.barrier()
        return None
    ndev = 1 if args.same_device else min(world, torch.cuda.device_count())
    gpu = K.GpuProfile(kv_bytes_per_token=L * pb // cfg["block_tokens"], num_layers=L, hbm_capacity=4 * n * pb)
    links = K.LinkProfile(network_bandwidth=NVLINK_PEAK_GBS * 1e9)
    cluster = K.PayloadCluster()
    stores, nodes = [], []
    for i in range(world):
        st = K.KvStore(gpu=gpu, links=links, opts=K.Options(node_id=i, write_behind=False, host_capacity=4 * n * pb))
        nd = K.NodePayload(cluster, i, K.PayloadOptions(
            device=i % ndev, num_kv_heads=cfg["kv_heads"], head_dim=cfg["head_dim"], dtype=kvx.BF16,
            device_pages=n, host_pages=1, landing_pages=2 * n, disk_pages=1, seed=0x70B, free_running=True,
            migrate_max_ctas=args.mig_ctas))
        nd.attach(st)
        for s_ in range(world):
            st.register_session(s_, f"ring{s_}")
        st.finalize_sessions()
        stores.append(st)
        nodes.append(nd)

    def pump(store, sched):
        for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
            store.apply_transfer(tid, at)

    now = 1_000_000
    for i in range(world):  # node i creates session i (K5 fill on its GPU)
        _, sched = stores[i].append_blocks(i, cfg["ctx"], now)
        pump(stores[i], sched)
    for nd in nodes:
        nd.synchronize()
    holder = list(range(world))  # holder[s] = node holding session s
    peer_streams = [torch.cuda.ExternalStream(nd.stream(K.LANE_PEER), device=torch.device("cuda", nd.opts.device))
                    for nd in nodes]

    def step(timed):
        nonlocal now
        now += 10_000_000_000
        evs = []
        for s_ in range(world):
            src = holder[s_]
            if timed:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(peer_streams[src])
                evs.append([src, e0])
        scheds = []
        own = []  # per session: an event right before its own pushes are posted
        for s_ in range(world):
            src, dst = holder[s_], (holder[s_] + 1) % world
            stores[src].mark_migrating_out(s_)
            if timed:
                e_own = torch.cuda.Event(enable_timing=True)
                e_own.record(peer_streams[src])
                own.append(e_own)
            scheds.append((dst, stores[dst].import_migration(s_, cfg["ctx"], now)))  # posts the 80 pushes
        for ev in evs:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(peer_streams[ev[0]])
            ev.append(e1)
        if timed:
            for ev, e_own in zip(evs, own):
                ev.append(e_own)
        for dst, sched in scheds:
            pump(stores[dst], sched)
        for s_ in range(world):
            stores[holder[s_]].release_session(s_, now + 1)
            holder[s_] = (holder[s_] + 1) % world
        for nd in nodes:
            nd.synchronize()
        if not timed:
            return None
        # (step start -> last push, own posting start -> last push) per device
        return [(e[1].elapsed_time(e[2]), e[3].elapsed_time(e[2])) for e in evs]

    for _ in range(max(1, args.warmup)):
        step(False)
    steps = max(1, min(args.steps, 10))
    n0 = kvx.launch_count()
    t0 = time.perf_counter()
    timings = [step(True) for _ in range(steps)]
    per_step = [max(t[0] for t in tt) for tt in timings]
    per_device_own = [max(t[1] for t in tt) for tt in timings]
    wall = (time.perf_counter() - t0) / steps
    launches = kvx.launch_count() - n0
    # What each node holds now is the session's creation content, bit for bit.
    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    import oracle.oracle as O  # checker only
    rng = np.random.default_rng(11)
    checked = 0
    for s_ in range(world):
        nd = nodes[holder[s_]]
        for _ in range(4):
            layer, block = int(rng.integers(L)), int(rng.integers(blocks))
            want = np.zeros((1, pb), np.uint8)
            O.fill_pages(want, pb, np.zeros(1, np.uint32), O.tags_array(s_, layer, block), 0x70B,
                         O.Layout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], 1), 1)
            got = nd.read_block(s_, layer, block, K.HOST, pb)
            assert got is not None and np.array_equal(got, want[0]), f"session {s_} layer {layer} block {block}"
            checked += 1
    del layout
    t_mig = statistics.mean(per_step)
    session_bytes = n * pb
    achieved = session_bytes / (t_mig * 1e-3) / GB
    dist.barrier()
    host = {f"node{i}": {k: round(v / 1e3 / L / (steps + max(1, args.warmup)), 2)
                         for k, v in nd.host_ns().items() if k in ("posted", "retired")}
            for i, nd in enumerate(nodes)}
    return dict(value=world * session_bytes / (t_mig * 1e-3) / GB, ms_per_step=t_mig,
                clocks={"note": "not sampled on the store path (one process drives every device)"},
                session_bytes=session_bytes, cfg=cfg, verified=True, serving=None,
                e2e={"value": world * session_bytes / wall / GB, "unit": UNIT, "h2d_bytes_per_step": world * 2 * n * 4,
                     "d2h_bytes_per_step": 0, "ms_per_step": 1e3 * wall,
                     "path": "per session: kvs_mark_migrating_out -> kvs_import_migration -> apply x L -> "
                             "kvs_release_session, host wall clock per ring step (all sessions)"},
                store_path={"devices": ndev, "nodes": world, "probe_pages_checked": checked,
                            "host_us_per_layer": host, "per_step_max_device_ms": per_step,
                            "per_session_from_own_posting_ms": per_device_own,
                            "device_side_gbs": session_bytes / (statistics.mean(per_device_own) * 1e-3) / GB,
                            "note": "one host thread posts every node's import in turn (the reference simulator "
                                    "is single-threaded): value counts from the step's start, "
                                    "device_side_gbs from each session's own posting"},
                roofline={"bound": "nvlink" if ndev > 1 else "hbm", "achieved": achieved,
                          "peak": NVLINK_PEAK_GBS if ndev > 1 else None, "unit": "GB/s",
                          "frac": achieved / NVLINK_PEAK_GBS if ndev > 1 else None, "traffic": None,
                          "frac_of_nominal_900": achieved / NVLINK_NOMINAL_GBS if ndev > 1 else None,
                          "peak_provenance": NVLINK_PEAK_PROVENANCE,
                          "kernel": "kvx_copy_pages (K3 push, store NetArrive)",
                          "algorithmic_bytes_per_launch": session_bytes // L,
                          "note": "per session per direction; the max over devices of the push sequence"},
                gpu_launches=launches)


def bench_multi(args, torch, np, kvx, dev, rank, world):
    """Migration-plus-serving at N GPUs (config 3): every rank decodes a batch
    of 70B @32K requests on its main stream while its own 70B @32K session
    migrates to rank (r+1) % N on a side stream — the reference's
    start_migration -> per-layer NetArrive (simcore.cpp:132-141,
    kvstore.cpp:753-769) as real bytes, off the serving path.

    --migrate-mode p2p (default): K3 (kvx_copy_pages) on the source GPU
      gathers the session's pages and stores them straight into the
      receiver's page pool over NVLink (opened through CUDA IPC): one pass,
      no staging buffer, no receiver-side kernel, no collective.
    --migrate-mode nccl: the comparison path through the C ABI —
      kvx_migrate_nccl: per layer K1 pack, ncclSend/ncclRecv around the ring
      (one group), K2 unpack on the receiver (gloo test mode: host-staged).

    value = N x session bytes / the max over ranks of the migration time
    measured WHILE decode runs. Also reported: the migration alone, the decode
    step alone and during the migration, and e2e (block tables H2D from
    pinned host every step, a probe page of what landed D2H)."""
    import torch.distributed as dist
    from paper_2412_16434_b200 import cluster
    cfg = dict(CFG_70B)
    if args.layers:
        cfg["layers"] = args.layers
    L = cfg["layers"]
    blocks, n = session_pages(cfg)
    layout = kvx.PageLayout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], kvx.BF16)
    pb = layout.page_bytes()
    pool = kvx.Pool(2 * n, pb, device=dev.index)
    src_ids, _ = cluster.session_layout(rank, 2 * n, n)
    d_src = torch.from_numpy(src_ids.view(np.int32)).to(dev)
    seed = cluster.session_seed(rank)

    def tags_for(seed_, count=n):
        layer = np.repeat(np.arange(L, dtype=np.uint32), blocks)[:count]
        block = np.tile(np.arange(blocks, dtype=np.uint32), L)[:count]
        return torch.from_numpy(np.stack([np.full(count, seed_, np.uint32), layer, block], -1).view(np.int32)).to(dev)

    kvx.fill_pages(pool, d_src, tags_for(seed), n, seed, layout, kvx.FILL_VALUES)
    nxt, prv = cluster.ring_peer(rank, world), cluster.ring_source(rank, world)
    _, my_dst = cluster.session_layout(rank, 2 * n, n)      # where my source's session lands in my pool
    _, peer_dst = cluster.session_layout(nxt, 2 * n, n)     # where mine lands in the receiver's pool
    d_my_dst = torch.from_numpy(my_dst.view(np.int32)).to(dev)
    d_peer_dst = torch.from_numpy(peer_dst.view(np.int32)).to(dev)
    mode = {"auto": kvx.COPY_AUTO, "sm": kvx.COPY_SM, "tma": kvx.COPY_TMA}[args.copy_mode]
    red_dev = dev if dist.get_backend() == "nccl" else None
    side = torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    sl = [slice(l * blocks, (l + 1) * blocks) for l in range(L)]

    peer = None
    if args.migrate_mode == "p2p":
        # Every rank opens its receiver's pool over CUDA IPC; if any rank
        # cannot (no peer access between these GPUs), all ranks agree to run
        # the NCCL path instead and the JSON says why.
        err = None
        try:
            peers = cluster.exchange_pool_handles(dist, rank, pool.ipc_export(), 2 * n, pb)
            if os.environ.get("BENCH_FAIL_IPC_RANK") == str(rank):  # test hook for the fallback below
                raise RuntimeError("peer open refused (BENCH_FAIL_IPC_RANK)")
            peer = kvx.Pool.ipc_open(peers[nxt].handle, peers[nxt].num_pages, pb, dev.index)
        except Exception as e:  # noqa: BLE001 — reported, and the bench continues over NCCL
            err = f"rank {rank}: {e}"[:200]
        errs = [None] * world
        dist.all_gather_object(errs, err)
        errs = [e for e in errs if e]
        if errs:
            if peer is not None:
                peer.close()
            peer = None
            args.migrate_mode = "nccl"
            args.p2p_unavailable = errs[0]

    if args.migrate_mode == "p2p":
        def migrate(st, src=d_src, dst=d_peer_dst):
            for l in range(L):
                kvx.copy_pages(pool, src[sl[l]], peer, dst[sl[l]], blocks, mode, st.cuda_stream,
                               max_ctas=args.mig_ctas)
    else:
        staged = dist.get_backend() != "nccl"  # gloo (CPU tests): host-staged send/recv
        bufs = [[torch.empty(blocks * pb, dtype=torch.uint8, device=dev) for _ in range(2)] for _ in range(2)]
        hbufs = [torch.empty(blocks * pb, dtype=torch.uint8) for _ in range(2)] if staged else None

        def migrate(st, src=d_src, dst=d_my_dst):
            with torch.cuda.stream(st):
                if staged:  # gloo (tests): host-staged, one layer at a time
                    for l in range(L):
                        snd, rcv = bufs[l % 2]
                        kvx.pack(pool, src[sl[l]], blocks, snd, kvx.COPY_AUTO, st.cuda_stream)
                        st.synchronize()
                        hbufs[0].copy_(snd)
                        ops = [dist.P2POp(dist.isend, hbufs[0], nxt), dist.P2POp(dist.irecv, hbufs[1], prv)]
                        for w in dist.batch_isend_irecv(ops):
                            w.wait()
                        rcv.copy_(hbufs[1])
                        kvx.unpack(pool, dst[sl[l]], blocks, rcv, kvx.COPY_AUTO, st.cuda_stream)
                    return
                # NCCL through the C ABI (kvx_migrate_nccl): per layer, K1 pack
                # -> one ncclSend/ncclRecv group around the ring -> K2 unpack,
                # on this side stream, over a communicator libkvx built.
                kvx.migrate_nccl(pool, src, n, nxt, pool, dst, n, prv, blocks, nccl_comm, nccl_staging,
                                 st.cuda_stream)

        nccl_comm, nccl_staging = None, None
        if not staged:
            uid = [kvx.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            nccl_comm = kvx.nccl_comm_init_rank(world, uid[0], rank, dev.index)
            nccl_staging = torch.empty(kvx.migrate_nccl_staging_bytes(pb, blocks), dtype=torch.uint8, device=dev)

    # Serving: a decode batch on every rank (70B shape: 64 q heads over 8 kv heads).
    B, hq = args.serve_batch, 64
    ctx = cfg["ctx"]
    dec_pages = B * L * blocks
    dpool = kvx.Pool(max(dec_pages, 1), pb, device=dev.index)
    if B:
        ids = torch.arange(dec_pages, dtype=torch.int32, device=dev)
        kvx.fill_pages(dpool, ids, torch.stack([ids * 0 + 1000 + rank, ids * 0, ids], -1).contiguous(), dec_pages,
                       7 + rank, layout, kvx.FILL_VALUES)
        perm = torch.randperm(dec_pages, device=dev, dtype=torch.int64).to(torch.int32)
        tables = [perm[l * B * blocks:(l + 1) * B * blocks].view(B, blocks).contiguous() for l in range(L)]
        ctx_t = torch.full((B,), ctx, dtype=torch.int32, device=dev)
        q = (torch.randn(B, hq, 128, device=dev) * 0.5).to(torch.bfloat16)
        out = torch.empty(B, hq, 128, dtype=torch.float32, device=dev)
        att = kvx.Attention(layout, hq, blocks, flags=DECODE_FLAGS(kvx))
        ws = torch.zeros(max(att.workspace_bytes(B, ctx), 1), dtype=torch.uint8, device=dev)

    def decode(st):
        for l in range(L):
            att(dpool, tables[l], ctx_t, q, out, B, ctx, ws, st.cuda_stream)

    def timed(fn, st):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(st)
        fn(st)
        e[1].record(st)
        return e

    torch.cuda.synchronize()
    dist.barrier()
    # Warm-up doubles as the calibration of the serving window: migration
    # alone and one decode step alone (every rank migrating at once).
    for _ in range(args.warmup):
        migrate(side)
    torch.cuda.synchronize()
    dist.barrier()
    em = timed(migrate, side)
    torch.cuda.synchronize()
    t_mig_alone = cluster.max_over_ranks(dist, em[0].elapsed_time(em[1]), red_dev)
    t_step = 0.0
    if B:
        decode(main)
        ed = timed(decode, main)
        torch.cuda.synchronize()
        t_step = cluster.max_over_ranks(dist, ed[0].elapsed_time(ed[1]), red_dev)
    # decode steps per migration: enough that the migration starts and ends inside the serving window
    K = max(1, int(np.ceil(1.25 * t_mig_alone / t_step))) if B else 0
    dist.barrier()

    rows = []
    n_launch0 = kvx.launch_count()
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            torch.cuda.synchronize()
            dist.barrier()
            e[0].record(main)
            side.wait_event(e[0])
            migrate(side)
            e[1].record(side)
            for _ in range(K):
                decode(main)
            e[2].record(main)
            torch.cuda.synchronize()
            rows.append((e[0].elapsed_time(e[1]), e[0].elapsed_time(e[2])))
        LAUNCHES["multi"] = kvx.launch_count() - n_launch0  # NCCL kernels are not counted (library)
        dist.barrier()  # every sender has finished writing into its receiver
    t_mig = cluster.max_over_ranks(dist, statistics.mean(r[0] for r in rows), red_dev)
    t_win = cluster.max_over_ranks(dist, statistics.mean(r[1] for r in rows), red_dev)

    # What landed here is the ring source's session, bit for bit.
    expect = kvx.Pool(n, pb, device=dev.index)
    kvx.fill_pages(expect, torch.arange(n, dtype=torch.int32, device=dev), tags_for(cluster.session_seed(prv)),
                   n, cluster.session_seed(prv), layout, kvx.FILL_VALUES)
    torch.cuda.synchronize()
    probe = torch.randint(0, n, (min(n, 4096),), device=dev)
    got = pool.as_tensor()[d_my_dst[probe].long()]
    ok = bool(torch.equal(got, expect.as_tensor()[probe]))
    expect.close()
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    assert all(oks), f"migrated pages differ on ranks {[i for i, o in enumerate(oks) if not o]}"

    gate = bench_multi_pipeline_gate(torch, np, kvx, dev, dist, cluster, pool, peer, d_src, d_peer_dst, d_my_dst,
                                     blocks, L, layout, red_dev, args.mig_ctas) if args.migrate_mode == "p2p" else None
    e2e = bench_multi_e2e(args, torch, np, kvx, dev, dist, cluster, pool, peer, src_ids, peer_dst, my_dst, pb, n,
                          blocks, red_dev) if args.migrate_mode == "p2p" else None

    session_bytes = n * pb
    value = world * session_bytes / (t_mig * 1e-3) / GB
    achieved = session_bytes / (t_mig * 1e-3) / GB  # per GPU per direction over NVLink
    serving = None
    if B:
        serving = {"decode": f"batch {B} x ctx {ctx} x {L} layers (K4, {hq} q / {cfg['kv_heads']} kv heads)",
                   "decode_step_ms_alone": t_step, "decode_steps_per_migration": K,
                   "window_ms": t_win, "decode_slowdown_over_window": t_win / (K * t_step) - 1.0,
                   "migration_inside_window": bool(t_mig <= t_win),
                   "migrate_ms_alone": t_mig_alone, "migrate_gbs_alone": session_bytes / (t_mig_alone * 1e-3) / GB}
    if peer is not None:
        peer.close()
    dist.barrier()
    launches_mine = LAUNCHES.get("multi", 0)
    per_rank = [None] * world
    dist.all_gather_object(per_rank, launches_mine)
    launches = int(sum(per_rank))  # every rank's libkvx launches in the timed loop (kvx_launch_count)
    if serving is not None and gate is not None:
        serving["pipeline_gate"] = gate
    return dict(value=value, ms_per_step=t_mig, clocks=clocks.summary(), session_bytes=session_bytes,
                cfg=cfg, verified=True, serving=serving, e2e=e2e,
                roofline={"bound": "nvlink", "achieved": achieved, "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                          "frac": achieved / NVLINK_PEAK_GBS, "traffic": None,
                          "frac_of_nominal_900": achieved / NVLINK_NOMINAL_GBS,
                          "peak_provenance": NVLINK_PEAK_PROVENANCE,
                          "kernel": "kvx_copy_pages(peer)" if args.migrate_mode == "p2p" else "nccl send/recv",
                          "algorithmic_bytes_per_launch": session_bytes // L,
                          "note": "per GPU, per direction, measured while decode runs; one launch per layer",
                          "peak_kind": "measured peer copy (B200_PROFILING.md)"},
                gpu_launches=launches)


def bench_multi_pipeline_gate(torch, np, kvx, dev, dist, cluster, pool, peer, d_src, d_peer_dst, d_my_dst, blocks,
                              L, layout, red_dev, mig_ctas=0):
    """The reference's layer-wise pipeline gate (pipeline_gate, kvstore.cpp:
    46-59; a request may decode layer l as soon as layer l has arrived)
    realised across GPUs with device-side signals, no host in the loop: after
    each layer's K3 launch the sender's stream writes the step number into
    the receiver's per-layer flag (kvx_signal_write into the receiver's flag
    page, opened through CUDA IPC); the receiver's decode of the migrating
    session (batch 1, 64 q heads, full context) waits on flag l
    (kvx_signal_wait) before attending over layer l. Compared with the
    recurrence's prediction from the measured per-layer arrivals and decode
    time, and with waiting for the whole session first."""
    from paper_2412_16434_b200 import kvstore as K
    rank, world = dist.get_rank(), dist.get_world_size()
    prv, nxt = cluster.ring_source(rank, world), cluster.ring_peer(rank, world)
    main, side = torch.cuda.current_stream(dev), torch.cuda.Stream(dev)
    fpb = (4 * L + 15) // 16 * 16
    flags = kvx.Pool(1, fpb, device=dev.index)
    flags.as_tensor().zero_()
    torch.cuda.synchronize()
    peers = cluster.exchange_pool_handles(dist, rank, flags.ipc_export(), 1, fpb)
    peer_flags = kvx.Pool.ipc_open(peers[nxt].handle, 1, fpb, dev.index)
    # Capability probe (every rank, then agree): stream memory ops on a
    # peer's IPC-mapped page. If any rank cannot, all skip the gate together.
    err = None
    try:
        kvx.signal_write(peer_flags.base, 0, side.cuda_stream)
        kvx.signal_wait(flags.base, 0, side.cuda_stream)
        side.synchronize()
    except Exception as e:  # noqa: BLE001 — reported in the JSON, not fatal to the bench
        err = str(e)
    errs = [None] * world
    dist.all_gather_object(errs, err)
    if any(errs):
        peer_flags.close()
        return {"skipped": f"device signals unavailable: {[e for e in errs if e][0]}"}
    sl = [slice(l * blocks, (l + 1) * blocks) for l in range(L)]
    tables = [d_my_dst[sl[l]].view(1, blocks) for l in range(L)]
    ctx = blocks * layout.block_tokens
    ctx_t = torch.full((1,), ctx, dtype=torch.int32, device=dev)
    q = (torch.randn(1, 64, 128, device=dev) * 0.5).to(torch.bfloat16)
    out = torch.empty(1, 64, 128, dtype=torch.float32, device=dev)
    att = kvx.Attention(layout, 64, blocks, flags=DECODE_FLAGS(kvx))
    ws = torch.zeros(max(att.workspace_bytes(1, ctx), 1), dtype=torch.uint8, device=dev)

    def send(step=None, timing=None):
        for l in range(L):
            kvx.copy_pages(pool, d_src[sl[l]], peer, d_peer_dst[sl[l]], blocks, kvx.COPY_AUTO, side.cuda_stream,
                           max_ctas=mig_ctas)
            if step is not None:
                kvx.signal_write(peer_flags.base + 4 * l, step, side.cuda_stream)
            if timing is not None:
                timing[l + 1].record(side)

    # measured alone: per-layer decode time, and the arrivals (sender clock)
    for l in range(L):
        att(pool, tables[l], ctx_t, q, out, 1, ctx, ws, main.cuda_stream)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(main)
    for l in range(L):
        att(pool, tables[l], ctx_t, q, out, 1, ctx, ws, main.cuda_stream)
    e[1].record(main)
    torch.cuda.synchronize()
    t_layer_us = e[0].elapsed_time(e[1]) * 1e3 / L
    dist.barrier()
    tev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
    tev[0].record(side)
    send(timing=tev)
    torch.cuda.synchronize()
    ready_us = [tev[0].elapsed_time(tev[l + 1]) * 1e3 for l in range(L)]
    all_ready = [None] * world
    dist.all_gather_object(all_ready, ready_us)
    src_ready = all_ready[prv]

    gated = []
    outs = [torch.empty(1, 64, 128, dtype=torch.float32, device=dev) for _ in range(L)]
    landing = d_my_dst.long()
    for step in range(1, 4):
        pool.as_tensor()[landing] = 0  # a decode that read a layer before it landed would see zeros
        torch.cuda.synchronize()
        dist.barrier()
        t = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        t[0].record(main)
        side.wait_event(t[0])
        send(step=step)
        for l in range(L):
            kvx.signal_wait(flags.base + 4 * l, step, main.cuda_stream)
            att(pool, tables[l], ctx_t, q, outs[l], 1, ctx, ws, main.cuda_stream)
        t[1].record(main)
        torch.cuda.synchronize()
        gated.append(t[0].elapsed_time(t[1]) * 1e3)
    dist.barrier()
    # The gated decode saw every layer only after it landed: same outputs as a
    # decode of the fully arrived session.
    plain = kvx.Attention(layout, 64, blocks)
    ref = torch.empty(1, 64, 128, dtype=torch.float32, device=dev)
    ok = True
    for l in range(L):
        plain(pool, tables[l], ctx_t, q, ref, 1, ctx, ws, main.cuda_stream)
        torch.cuda.synchronize()
        ok = ok and bool(torch.equal(ref, outs[l]))
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    assert all(oks), f"gated decode read a layer before it arrived on ranks {[i for i, o in enumerate(oks) if not o]}"
    peer_flags.close()
    measured = statistics.median(gated)
    first_end, _, stall = K.pipeline_gate([int(r * 1e3) for r in src_ready], 0, int(L * t_layer_us * 1e3))
    worst = cluster.max_over_ranks(dist, measured, red_dev)
    return {"decode": f"batch 1 over the migrating session ({L} layers, ctx {ctx}, 64 q heads)",
            "layer_arrival_us_first_last": [src_ready[0], src_ready[-1]], "layer_decode_us": t_layer_us,
            "measured_first_step_end_us": measured, "max_over_ranks_us": worst,
            "predicted_first_step_end_us": first_end / 1e3, "predicted_stall_us": stall / 1e3,
            "unpipelined_us": src_ready[-1] + L * t_layer_us, "mover_max_ctas": mig_ctas or "all",
            "outputs_verified": True,
            "how": "per-layer device flags: sender stream writes into the receiver's flag page over IPC after "
                   "each K3 launch (kvx_signal_write), receiver stream waits on it before each K4 (kvx_signal_wait)"}


def bench_multi_e2e(args, torch, np, kvx, dev, dist, cluster, pool, peer, src_ids, peer_dst, my_dst, pb, n,
                    blocks, red_dev):
    """Migration end to end between HOST tiers, as the reference models it
    (the source's copy moves to the receiver, which lands it in its HOST tier:
    NetArrive sets kHost, kvstore.cpp:914-923). Per step and per layer, with
    the session's first `layers` layers (a bounded sample: pinned host buffers
    for a whole 70B session on every rank would not fit the host):
      source: pinned HOST -> H2D staging -> K2 unpack into its DEVICE pages ->
              K3 into the receiver's pool over NVLink (CUDA IPC);
      (every rank's sends landed: barrier)
      receiver: K1 pack of what landed -> D2H -> pinned HOST.
    Streams per direction overlap layers; max over ranks; bytes verified."""
    L = min(8, n // blocks)
    lb = blocks * pb
    rank, world = dist.get_rank(), dist.get_world_size()
    prv = cluster.ring_source(rank, world)
    g = torch.Generator().manual_seed(1000 + rank)
    h_src = torch.randint(0, 256, (L * lb,), dtype=torch.uint8, generator=g).pin_memory()
    h_dst = torch.empty(L * lb, dtype=torch.uint8).pin_memory()
    NB = 3
    stage = [torch.empty(lb, dtype=torch.uint8, device=dev) for _ in range(NB)]
    s_in, s_c, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    main = torch.cuda.current_stream(dev)
    d_src = torch.from_numpy(src_ids.view(np.int32)).to(dev)
    d_peer = torch.from_numpy(peer_dst.view(np.int32)).to(dev)
    d_mine = torch.from_numpy(my_dst.view(np.int32)).to(dev)

    def send_phase():
        s_in.wait_stream(main)
        done = {}
        for l in range(L):
            sl = slice(l * blocks, (l + 1) * blocks)
            with torch.cuda.stream(s_in):
                if l - NB in done:
                    s_in.wait_event(done.pop(l - NB))
                stage[l % NB].copy_(h_src[l * lb:(l + 1) * lb], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
            s_c.wait_event(e)
            kvx.unpack(pool, d_src[sl], blocks, stage[l % NB], kvx.COPY_AUTO, s_c.cuda_stream)
            kvx.copy_pages(pool, d_src[sl], peer, d_peer[sl], blocks, kvx.COPY_AUTO, s_c.cuda_stream)
            e2 = torch.cuda.Event()
            e2.record(s_c)
            done[l] = e2
        main.wait_stream(s_c)

    def receive_phase():
        s_c.wait_stream(main)
        done = {}
        for l in range(L):
            sl = slice(l * blocks, (l + 1) * blocks)
            if l - NB in done:
                s_c.wait_event(done.pop(l - NB))
            kvx.pack(pool, d_mine[sl], blocks, stage[l % NB], kvx.COPY_AUTO, s_c.cuda_stream)
            e = torch.cuda.Event()
            e.record(s_c)
            with torch.cuda.stream(s_out):
                s_out.wait_event(e)
                h_dst[l * lb:(l + 1) * lb].copy_(stage[l % NB], non_blocking=True)
                e2 = torch.cuda.Event()
                e2.record(s_out)
                done[l] = e2
        main.wait_stream(s_out)

    def step():
        send_phase()
        torch.cuda.synchronize()
        dist.barrier()  # every sender's pages have landed in its receiver
        receive_phase()

    step()
    torch.cuda.synchronize()
    dist.barrier()
    steps = max(1, min(args.steps, 3))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(main)
    for _ in range(steps):
        step()
    e[1].record(main)
    torch.cuda.synchronize()
    ms = cluster.max_over_ranks(dist, e[0].elapsed_time(e[1]) / steps, red_dev)
    dist.barrier()
    expect = torch.randint(0, 256, (L * lb,), dtype=torch.uint8, generator=torch.Generator().manual_seed(1000 + prv))
    ok = bool(torch.equal(h_dst, expect))
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    assert all(oks), f"e2e HOST-to-HOST bytes differ on ranks {[i for i, o in enumerate(oks) if not o]}"
    return {"value": world * L * lb / (ms * 1e-3) / GB, "unit": UNIT, "h2d_bytes_per_step": L * lb,
            "d2h_bytes_per_step": L * lb, "ms_per_step": ms, "steps": steps, "layers_sampled": L,
            "path": "source pinned HOST -> H2D -> kvx_unpack -> kvx_copy_pages into the peer pool (IPC/NVLink) | "
                    "barrier | receiver kvx_pack -> D2H -> pinned HOST (per layer, streams overlap layers)"}


# ---------------------------------------------------------------------------
# CPU side (oracle; test infrastructure only, used here as the reported baseline)


def cpu_migrate(np, cfg, seconds_budget, layers=None, repeat_min=1):
    """Payload restatement pack+unpack (OpenMP, all host threads)."""
    import oracle.oracle as O
    blocks, n = session_pages(cfg)
    L = layers or cfg["layers"]
    n = L * blocks
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    rng = np.random.default_rng(7)
    perm = rng.permutation(2 * n).astype(np.uint32)
    pool = np.zeros((2 * n, pb), np.uint8)
    buf = np.empty(n * pb, np.uint8)
    lay = O.Layout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], 1)
    tags = O.tags_array(0, np.repeat(np.arange(L), blocks), np.tile(np.arange(blocks), L))
    O.fill_pages(pool, pb, perm[:n], tags, 1, lay, 0)
    reps, t_total = 0, 0.0
    while reps < repeat_min or t_total < seconds_budget:
        t0 = time.perf_counter()
        O.pack(pool, pb, perm[:n], buf)
        O.unpack(pool, pb, perm[n:2 * n], buf)
        t_total += time.perf_counter() - t0
        reps += 1
    assert np.array_equal(pool[perm[n]], pool[perm[0]])
    return n * pb * reps / t_total / GB, O.threads(), f"{L} layers x {blocks} pages x {pb} B, {reps} reps"


def reference_state_ops(np):
    """The reference KvStore's bookkeeping for one migrated 8B@8K session."""
    from paper_2412_16434_b200 import kvstore as K
    import oracle.oracle as O
    if not O.REF_KVS_LIB.exists():
        return None
    cfg = CFG_8B
    gpu = K.GpuProfile(kv_bytes_per_token=cfg["layers"] * 4096, num_layers=cfg["layers"],
                       hbm_capacity=180_000_000_000)
    st = K.KvStore(gpu=gpu, lib=str(O.REF_KVS_LIB))
    st.register_session(0, "s0")
    st.finalize_sessions()
    t0 = time.perf_counter()
    sched = st.import_migration(0, cfg["ctx"], 0)
    for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
        st.apply_transfer(tid, at)
    st.release_session(0, 0)
    return time.perf_counter() - t0


def arm_config(cfg, world, path="store"):
    """The workload both arms report (identical for --impl b200 / reference)."""
    blocks, n = session_pages(cfg)
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    if world == 1:
        workload = (f"{cfg['model']} @{cfg['ctx']} session ({cfg['layers']} layers x {blocks} pages): pack every "
                    "page into the migration buffer + unpack into a second page permutation")
    elif path == "store":
        workload = (f"{cfg['model']} @{cfg['ctx']} session per node, every session migrated one hop around the "
                    "ring per step through the store API (mark_migrating_out -> import_migration -> apply every "
                    "NetArrive -> release)")
    else:
        workload = (f"{cfg['model']} @{cfg['ctx']} session per rank, ring migration rank r -> r+1 "
                    "(page-to-page into the receiver's pool) while every rank decodes a batch of 4 "
                    f"{cfg['model']} @{cfg['ctx']} requests")
    return {"workload": workload, "kv_shape": cfg["model"], "seq_len": cfg["ctx"], "layers": cfg["layers"],
            "kv_heads": cfg["kv_heads"], "head_dim": cfg["head_dim"], "kv_dtype": "bf16", "page_bytes": pb,
            "session_bytes": n * pb, "parallelism": "single" if world == 1 else f"ring-p2p{world}",
            "l2": "inputs larger than the 126 MB L2 (1 GiB / 10.7 GB per step); no flush"}


def run_reference(args):
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    # torchrun sets OMP_NUM_THREADS=1 per rank; the reference arm runs on rank
    # 0 alone and may use every host core (set before OpenMP initialises).
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    cfg = CFG_8B if world == 1 else CFG_70B
    import oracle.oracle as O
    O.build_payload()
    blocks, n = session_pages(cfg)
    layers = cfg["layers"] if world == 1 else 8  # 70B: bounded sample of 8 layers (2.7 GB)
    pb = 2 * cfg["kv_heads"] * cfg["block_tokens"] * cfg["head_dim"] * 2
    nb = layers * blocks
    rng = np.random.default_rng(7)
    perm = rng.permutation(2 * nb).astype(np.uint32)
    pool = np.zeros((2 * nb, pb), np.uint8)
    buf = np.empty(nb * pb, np.uint8)
    lay = O.Layout(cfg["kv_heads"], cfg["head_dim"], cfg["block_tokens"], 1)
    O.fill_pages(pool, pb, perm[:nb], O.tags_array(0, np.repeat(np.arange(layers), blocks),
                                                   np.tile(np.arange(blocks), layers)), 1, lay, 0)
    state_s = 0.0

    def step():
        nonlocal state_s
        s = reference_state_ops(np)
        state_s += s or 0.0
        O.pack(pool, pb, perm[:nb], buf)
        O.unpack(pool, pb, perm[nb:2 * nb], buf)

    for _ in range(args.warmup):
        step()
    state_s = 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = nb * pb * args.steps / dt / GB
    threads = O.threads()
    sample = (f"{layers} of {cfg['layers']} layers x {blocks} pages x {pb} B per step: reference KvStore "
              f"import_migration+apply+release (oracle/_ref, 1 thread, {1e3 * state_s / args.steps:.2f} ms/step) "
              f"+ payload pack/unpack restatement (OpenMP {threads} threads)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": arm_config(cfg, world, args.path),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--copy-mode", default="auto", choices=["auto", "sm", "tma"])
    ap.add_argument("--skip-attention", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-overlap", action="store_true")
    ap.add_argument("--attn-sweep", action="store_true", help="diagnostic: time fixed split-K factors")
    ap.add_argument("--bg-sweep", action="store_true", help="diagnostic: sweep mover CTA caps beside decode")
    ap.add_argument("--bg-batch", type=int, default=16, help="decode batch of the overlap / background section")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"], help="N>1 control plane")
    ap.add_argument("--same-device", action="store_true", help="test mode: all ranks on cuda:0")
    ap.add_argument("--layers", type=int, default=0, help="test mode: shrink the N>1 session")
    ap.add_argument("--migrate-mode", default="p2p", choices=["p2p", "nccl"],
                    help="N>1: K3 stores into the peer pool (p2p) or pack + send/recv + unpack (nccl)")
    ap.add_argument("--mig-ctas", type=int, default=0, help="N>1: cap on the migration mover's CTAs (0 = all)")
    ap.add_argument("--serve-batch", type=int, default=4, help="N>1: decode batch run beside the migration")
    ap.add_argument("--path", default="store", choices=["store", "kvx"],
                    help="N>1: store = migrations through the store API (KvStore + NodePayload, one process "
                         "driving every device: the product path); kvx = raw K3 ring over CUDA IPC with decode "
                         "beside it (one process per GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    from paper_2412_16434_b200 import kvx

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:  # test mode: every rank on cuda:0 (IPC between processes, one GPU)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    kvx.lib()
    hbm_peak, peak_kind = load_peaks()

    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        if args.path == "store":
            res = bench_store_ring(args, torch, np, kvx, rank, world)
        else:
            res = bench_multi(args, torch, np, kvx, dev, rank, world)
        cfg = res["cfg"] if res is not None else None
    else:
        res = bench_single(args, torch, np, kvx, dev, hbm_peak, peak_kind)
        cfg = CFG_8B

    if rank == 0:
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": arm_config(cfg, world, args.path),
                "roofline": res["roofline"], "clocks": res["clocks"], "gpu_launches": res["gpu_launches"]}
        if world > 1:
            line["serving"] = res["serving"]
            if res["e2e"] is not None:
                line["e2e"] = res["e2e"]
            line["config"]["migrate_mode"] = args.migrate_mode if args.path == "kvx" else "store-api"
            line["config"]["path"] = args.path
            if "store_path" in res:
                line["store_path"] = res["store_path"]
            if getattr(args, "p2p_unavailable", None):
                line["config"]["p2p_unavailable"] = args.p2p_unavailable
        if world == 1:
            line["e2e"] = res["e2e"]
            line["decode_attention"] = res["attention"]
            line["overlap"] = res["overlap"]
            line["store_cycle"] = res["store_cycle"]
            line["disk_tier"] = res["disk_tier"]
            line["detail"] = res["extra"]
            if not args.skip_cpu:
                v, cores, sample = cpu_migrate(np, cfg, 8.0, layers=8, repeat_min=3)
                line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                        "sample": f"oracle pack+unpack, {sample}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
