"""CPU-side checks of the kvx C ABI library (no kernels launched here)."""
import ctypes
import re

import pytest

from conftest import ROOT


def test_kvx_library_exports_every_declared_symbol(product_libs):
    decl = (ROOT / "include" / "kvx.h").read_text()
    names = re.findall(r"^\s*(?:int|void\*?|uint64_t|const char\*)\s*\*?\s*(kvx_\w+)\(", decl, re.M)
    assert len(names) >= 20
    lib = ctypes.CDLL(str(product_libs.KVX_LIB))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing


def test_kvx_fails_loudly_without_a_device(product_libs):
    """No CPU fallback: pool creation must error when no CUDA device exists."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2412_16434_b200 import kvx
    with pytest.raises(kvx.KvxError):
        kvx.Pool(4, 4096, device=0)


def test_page_bytes_match_the_store_accounting(product_libs):
    """kvx page size == the reference's layer_block_bytes for each config
    (kvstore.cpp:67 = kv_bytes_per_layer(16) with kv_bytes_per_token summed
    over layers): tiny 2 L x 4 H x d64 fp32; 8B 32 L x 8 H x d128 bf16; 70B 80 L."""
    from paper_2412_16434_b200 import kvstore as K
    from paper_2412_16434_b200 import kvx
    for layers, heads, dim, dtype, elt in [(2, 4, 64, kvx.F32, 4), (32, 8, 128, kvx.BF16, 2),
                                           (80, 8, 128, kvx.BF16, 2)]:
        per_token = layers * 2 * heads * dim * elt
        gpu = K.GpuProfile(kv_bytes_per_token=per_token, num_layers=layers)
        assert K.kv_bytes_per_layer(16, gpu) == kvx.page_bytes(kvx.PageLayout(heads, dim, 16, dtype))


def test_file_pool_without_a_device(product_libs, tmp_path):
    """The DISK-tier file pool is host-only: creating it and reading a page
    needs no GPU (a fresh file reads as zeros); it refuses kernels."""
    from paper_2412_16434_b200 import kvx
    pb = 32768
    pool = kvx.Pool.file(tmp_path / "disk.pages", 8, pb)
    assert (tmp_path / "disk.pages").stat().st_size == 8 * pb
    assert not pool.read_page(7).any()
    with pytest.raises(kvx.KvxError):
        pool.read_page(8)
    with pytest.raises(kvx.KvxError):
        kvx.Pool.file(tmp_path / "bad.pages", 8, 1000)  # pages must be 4 KiB multiples (O_DIRECT)
    pool.close()


def test_kvx_library_loads_without_a_driver(product_libs):
    """libkvx.so resolves driver-API entry points through the runtime, so it
    has no hard dependency on libcuda.so (the build check and the CPU suite
    load it on machines without a GPU driver)."""
    import shutil
    import subprocess
    if shutil.which("readelf") is None:
        pytest.skip("readelf not available")
    out = subprocess.run(["readelf", "-d", str(product_libs.KVX_LIB)], capture_output=True, text=True).stdout
    assert "libcuda.so" not in out


def test_product_path_does_not_route_through_the_oracle(product_libs):
    """The oracle is test infrastructure: no product module imports it, no
    product library links it, and the store mirror loads the product library
    unless a test passes the oracle's path explicitly."""
    import ast
    import shutil
    import subprocess
    pkg = ROOT / "paper_2412_16434_b200"
    for py in pkg.glob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), py
            if isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", py
    if shutil.which("readelf"):
        for lib in (product_libs.KVX_LIB, product_libs.HOST_LIB):
            out = subprocess.run(["readelf", "-d", str(lib)], capture_output=True, text=True).stdout
            assert "oracle" not in out and "symsim_oracle" not in out, lib
    from paper_2412_16434_b200 import _build, kvstore as K
    lib = K.load_kvs_library()
    assert lib._name == str(_build.HOST_LIB) and "oracle" not in lib._name


def test_abi_rejects_bad_arguments_without_touching_a_device(product_libs):
    """Argument checks come before any CUDA call: null pools / ids, bad page
    sizes and bad layouts return KVX_ERR_ARG with a message (no crash, no
    device needed)."""
    lib = ctypes.CDLL(str(product_libs.KVX_LIB))
    lib.kvx_last_error.restype = ctypes.c_char_p
    V, U64 = ctypes.c_void_p, ctypes.c_uint64
    lib.kvx_copy_pages.argtypes = [V, V, V, V, U64, ctypes.c_int, V]
    lib.kvx_pack.argtypes = [V, V, U64, V, ctypes.c_int, V]
    lib.kvx_pool_create_host.argtypes = [U64, U64, ctypes.POINTER(V)]
    lib.kvx_signal_write.argtypes = [V, ctypes.c_uint32, V]
    KVX_ERR_ARG = 2
    assert lib.kvx_copy_pages(None, None, None, None, 4, 0, None) == KVX_ERR_ARG
    assert b"null" in lib.kvx_last_error()
    assert lib.kvx_pack(None, None, 1, None, 0, None) == KVX_ERR_ARG
    out = V()
    assert lib.kvx_pool_create_host(4, 1000, ctypes.byref(out)) == KVX_ERR_ARG  # not a multiple of 16
    assert lib.kvx_signal_write(V(2), 1, None) == KVX_ERR_ARG  # misaligned flag
    lib.kvx_copy_pages_listed.argtypes = [V, V, V, V, U64, ctypes.c_int, ctypes.c_uint32, V]
    assert lib.kvx_copy_pages_listed(None, None, None, None, 4, 0, 0, None) == KVX_ERR_ARG
    assert b"null" in lib.kvx_last_error()


def test_migrate_nccl_validates_arguments_before_touching_a_device(product_libs):
    """kvx_migrate_nccl (K3 over NCCL, include/kvx.h): argument errors are
    reported as KVX_ERR_ARG before NCCL or CUDA is touched; an empty call is
    a no-op; the staging size is 2 slots of one chunk."""
    import ctypes as C
    lib = C.CDLL(str(product_libs.KVX_LIB))
    lib.kvx_migrate_nccl.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_uint64, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
    lib.kvx_migrate_nccl_staging_bytes.restype = C.c_uint64
    lib.kvx_migrate_nccl_staging_bytes.argtypes = [C.c_uint64, C.c_uint64]
    assert lib.kvx_migrate_nccl_staging_bytes(65536, 512) == 2 * 65536 * 512
    assert lib.kvx_migrate_nccl(None, None, 0, -1, None, None, 0, -1, 16, None, None, 0, None) == 0
    fake = C.c_void_p(0x1000)
    # pages to send but no pool / ids / comm
    assert lib.kvx_migrate_nccl(None, None, 4, 1, None, None, 0, -1, 16, fake, fake, 1 << 30, None) == 2
    assert lib.kvx_migrate_nccl(fake, fake, 4, 1, None, None, 0, -1, 16, None, fake, 1 << 30, None) == 2
    assert lib.kvx_migrate_nccl(fake, fake, 4, -1, None, None, 0, -1, 16, fake, fake, 1 << 30, None) == 2
    assert lib.kvx_migrate_nccl(fake, fake, 4, 1, None, None, 0, -1, 0, fake, fake, 1 << 30, None) == 2
