"""K7 (skinny_linear): the decode step's projections at small batch, against a
plain PyTorch fp32 reference of the same op (Y (+)= X . W^T, bf16 in/out).

The serving engine's quanta (kvx_model_decode_step) run every projection of
a Llama-3.1-8B-shaped layer through kvx_model_linear's path: K7 for batch
rows <= 8, cuBLAS above. Checked here on every projection shape of the
model (QKV, O, gate/up, down, LM head) at rows 1..16 and past the K7 limit,
with and without the residual accumulate, within bf16 output rounding."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


class ModelConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("hidden", C.c_int32), ("num_q_heads", C.c_int32),
                ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("intermediate", C.c_int32),
                ("vocab", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_float)]


@pytest.fixture(scope="module")
def model():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_16434_b200 import kvx
    lib = kvx.lib()
    lib.kvx_model_create.argtypes = [C.c_int, C.POINTER(ModelConfig), C.c_uint64, C.POINTER(C.c_void_p)]
    lib.kvx_model_destroy.argtypes = [C.c_void_p]
    lib.kvx_model_linear.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_int32, C.c_void_p]
    # Llama-3.1-8B layer shapes, one layer, a small vocabulary (the LM head's
    # shape class is the same; the test needs no 1 GB embedding).
    cfg = ModelConfig(1, 4096, 32, 8, 128, 14336, 2048, 1e-5, 500000.0)
    m = C.c_void_p()
    assert lib.kvx_model_create(0, C.byref(cfg), 7, C.byref(m)) == 0, lib.kvx_last_error()
    yield lib, m
    lib.kvx_model_destroy(m)


SHAPES = [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096), (4096, 2048)]


@pytest.mark.parametrize("rows", [1, 3, 8, 9, 16, 17, 64])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_projection_matches_fp32_reference(model, rows, accumulate):
    import torch
    lib, m = model
    g = torch.Generator(device="cuda").manual_seed(rows * 10 + accumulate)
    st = torch.cuda.current_stream()
    for k, n in SHAPES:
        x = (torch.rand(rows, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        w = ((torch.rand(n, k, device="cuda", generator=g) * 2 - 1) / k ** 0.5).to(torch.bfloat16)
        y0 = (torch.rand(rows, n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        y = y0.clone()
        rc = lib.kvx_model_linear(m, x.data_ptr(), w.data_ptr(), y.data_ptr(), rows, k, n, accumulate,
                                  C.c_void_p(st.cuda_stream))
        assert rc == 0, lib.kvx_last_error()
        torch.cuda.synchronize()
        xw = x.float() @ w.float().t()
        ref = xw + y0.float() if accumulate else xw
        err = (y.float() - ref).abs()
        # bf16 output rounding (2^-8 relative) + fp32 summation-order noise;
        # accumulating, cuBLAS (rows > 16) may round X.W^T to bf16 before
        # adding Y: a second rounding of |X.W^T|.
        tol = 2 ** -8 * (ref.abs() + (xw.abs() if accumulate else 0)) + 1e-3 * ref.abs().max()
        assert bool((err <= tol).all()), (k, n, rows, accumulate, float(err.max()), float((err - tol).max()))


def test_projection_split_counters_reset(model):
    """Back-to-back launches on one stream reuse the split-K arrival counters:
    the same call twice gives bit-identical results (deterministic merge)."""
    import torch
    lib, m = model
    st = torch.cuda.current_stream()
    x = torch.randn(4, 14336, device="cuda").to(torch.bfloat16)
    w = (torch.randn(4096, 14336, device="cuda") / 120).to(torch.bfloat16)
    ys = []
    for _ in range(3):
        y = torch.zeros(4, 4096, device="cuda", dtype=torch.bfloat16)
        assert lib.kvx_model_linear(m, x.data_ptr(), w.data_ptr(), y.data_ptr(), 4, 14336, 4096, 0,
                                    C.c_void_p(st.cuda_stream)) == 0
        ys.append(y)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[1], ys[2])
