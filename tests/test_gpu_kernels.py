"""GPU kernel checks: the tcgen05 stream-K GEMM against a float64 host reference, its fused
epilogues, and batch invariance (a token column is bitwise identical for every padded token count)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bf16(x: np.ndarray) -> np.ndarray:
    """round-to-nearest-even to bf16, returned as uint16 bits"""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


def f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def gemm(epi, W, X, tp, n_valid=None, io=None):
    import ctypes as C
    from paper_2601_05524_b200 import _capi
    n_out, K = W.shape
    T = X.shape[0]
    cols = n_out // 2 if epi == 2 else n_out
    io = np.zeros((T, cols), np.float32) if io is None else np.ascontiguousarray(io, np.float32).copy()
    am = np.zeros(T, np.int32)
    W = np.ascontiguousarray(W)
    X = np.ascontiguousarray(X)
    _capi.check(_capi.lib().dbl_debug_gemm(
        epi, W.ctypes.data_as(C.POINTER(C.c_uint16)), n_out, K, X.ctypes.data_as(C.POINTER(C.c_uint16)),
        T, tp, n_valid if n_valid is not None else n_out, io.ctypes.data_as(C.POINTER(C.c_float)),
        am.ctypes.data_as(C.POINTER(C.c_int32))))
    return io, am


SHAPES = [(128, 64, 1), (256, 4096, 7), (512, 1024, 16), (7168, 5120, 5), (1024, 17408, 33), (384, 2048, 100)]


@pytest.mark.parametrize("n_out,K,T", SHAPES)
def test_gemm_store_f32_matches_float64(n_out, K, T):
    rng = np.random.default_rng(n_out + K + T)
    W = bf16(rng.standard_normal((n_out, K)) * 0.02)
    X = bf16(rng.standard_normal((T, K)))
    tp = max(16, -(-T // 16) * 16)
    got, _ = gemm(4, W, X, tp)
    ref = f32(X).astype(np.float64) @ f32(W).astype(np.float64).T
    err = np.abs(got - ref).max() / (np.abs(ref).max() + 1e-30)
    assert err < 2e-5, err


@pytest.mark.parametrize("n_out,K", [(7168, 5120), (256, 4096), (1024, 17408)])
def test_gemm_batch_invariance(n_out, K):
    """Columns computed inside a 16-, 48-, 112- and 256-token forward are bitwise identical."""
    rng = np.random.default_rng(7)
    W = bf16(rng.standard_normal((n_out, K)) * 0.02)
    X = bf16(rng.standard_normal((256, K)))
    base, _ = gemm(4, W, X[:1], 16)
    for tp, T in ((16, 9), (48, 40), (112, 100), (256, 256)):
        got, _ = gemm(4, W, X[:T], tp)
        assert np.array_equal(got[0], base[0]), tp
    full, _ = gemm(4, W, X, 256)
    part, _ = gemm(4, W, X[:37], 48)
    assert np.array_equal(full[:37], part)


def test_gemm_epilogues():
    rng = np.random.default_rng(3)
    n_out, K, T = 1024, 2048, 20
    W = bf16(rng.standard_normal((n_out, K)) * 0.02)
    X = bf16(rng.standard_normal((T, K)))
    ref = f32(X).astype(np.float64) @ f32(W).astype(np.float64).T
    # bf16 store
    got, _ = gemm(0, W, X, 32)
    assert np.abs(got - ref).max() <= np.abs(ref).max() * 2 ** -7
    # residual add
    resid = rng.standard_normal((T, n_out)).astype(np.float32)
    got, _ = gemm(1, W, X, 32, io=resid)
    assert np.abs(got - (resid + ref)).max() < 1e-4
    # SiLU(gate) * up with rows interleaved 16 gate | 16 up per 32
    got, _ = gemm(2, W, X, 32)
    r = ref.reshape(T, n_out // 32, 2, 16)
    g, u = r[:, :, 0, :].reshape(T, -1), r[:, :, 1, :].reshape(T, -1)
    want = g / (1 + np.exp(-g)) * u
    assert np.abs(got - want).max() <= np.abs(want).max() * 2 ** -6
    # argmax (lowest index on ties) with a partial last tile masked by n_valid
    n_valid = 1000
    logits, am = gemm(3, W, X, 32, n_valid=n_valid)
    assert np.array_equal(am, np.argmax(logits[:, :n_valid], axis=1))
    assert np.abs(logits[:, :n_valid] - ref[:, :n_valid]).max() < 2e-5 * np.abs(ref).max()


def test_gemm_argmax_ties_lowest_index():
    K = 64
    W = np.zeros((384, K), np.uint16)
    W[[5, 77, 300], 0] = bf16(np.array([1.0, 1.0, 1.0]))
    X = np.zeros((3, K), np.uint16)
    X[:, 0] = bf16(np.array([1.0, 1.0, 1.0]))
    _, am = gemm(3, W, X, 16)
    assert am.tolist() == [5, 5, 5]
