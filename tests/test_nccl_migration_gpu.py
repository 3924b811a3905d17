"""K3 over NCCL through the C ABI (kvx_migrate_nccl): two processes on two
GPUs, each holding a session in its pool, exchange them around a 2-ring
(pack -> ncclSend/ncclRecv -> unpack per layer) over a communicator libkvx
builds; each receiver checks what landed bit-exact. NCCL needs distinct
GPUs, so this skips on a one-GPU box (bench.py --migrate-mode nccl runs the
same call at N GPUs)."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from paper_2412_16434_b200 import kvx
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("gloo")
layout = kvx.PageLayout(8, 128, 16, kvx.BF16)
pb, blocks, layers = layout.page_bytes(), 64, 4
n = blocks * layers
pool = kvx.Pool(2 * n, pb, device=rank)
src = torch.arange(n, dtype=torch.int32, device=dev)
dst = torch.arange(n, 2 * n, dtype=torch.int32, device=dev).flip(0).contiguous()
tags = torch.stack([src * 0 + 100 + rank, src // blocks, src % blocks], -1).int().contiguous()
kvx.fill_pages(pool, src, tags, n, 5, layout, kvx.FILL_VALUES)
uid = [kvx.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = kvx.nccl_comm_init_rank(world, uid[0], rank, rank)
staging = torch.empty(kvx.migrate_nccl_staging_bytes(pb, blocks), dtype=torch.uint8, device=dev)
nxt, prv = (rank + 1) % world, (rank - 1) % world
kvx.migrate_nccl(pool, src, n, nxt, pool, dst, n, prv, blocks, comm, staging)
torch.cuda.synchronize()
ref = kvx.Pool(n, pb, device=rank)
rtags = torch.stack([src * 0 + 100 + prv, src // blocks, src % blocks], -1).int().contiguous()
kvx.fill_pages(ref, src, rtags, n, 5, layout, kvx.FILL_VALUES)
torch.cuda.synchronize()
ok = torch.equal(pool.as_tensor()[dst.long()], ref.as_tensor())
kvx.nccl_comm_destroy(comm)
print("OK" if ok else "MISMATCH", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_ring_exchange_bit_exact(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("NCCL p2p needs two GPUs")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, "ROOT": str(ROOT)})
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    assert proc.stdout.count("OK") == 2
