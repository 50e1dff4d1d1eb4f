"""Kernel-level checks of the Level-3 GEMM family behind the blocked sweeps (DMMA fp64,
tcgen05 kind::tf32 fp32, cp.async fallbacks) through cd_debug_gemm, against torch
(cuBLAS) matmul in fp64: every transpose combination, ragged sizes, split-K."""
import ctypes

import pytest
import torch

import paper_1602_07527_b200 as cd

pytestmark = pytest.mark.gpu


def run_gemm(A, B, C, ta, tb, alpha, beta):
    L = cd.lib()
    f = L.cd_debug_gemm
    f.argtypes = [ctypes.c_int] + [ctypes.c_int64] * 3 + [ctypes.c_int] * 2 + [ctypes.c_void_p, ctypes.c_int64] * 3 + \
        [ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    es = C.element_size()
    ws = torch.empty(304 * 128 * 128 * es, dtype=torch.uint8, device="cuda")
    M, N = C.shape
    K = A.shape[0] if ta else A.shape[1]
    dt = 0 if C.dtype == torch.float64 else 1
    rc = f(dt, M, N, K, ta, tb, A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), C.data_ptr(), C.stride(1),
           alpha, beta, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()


def colmajor(r, c, dtype):
    return torch.randn(c, r, dtype=dtype, device="cuda").t()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (200, 136, 72), (64, 300, 1000), (257, 129, 40), (300, 64, 200),
                                   (129, 40, 96), (512, 33, 64)])
def test_gemm_layouts(dtype, ta, tb, M, N, K):
    torch.manual_seed(M * 7 + N + K)
    A = colmajor(K, M, dtype) if ta else colmajor(M, K, dtype)
    B = colmajor(N, K, dtype) if tb else colmajor(K, N, dtype)
    C = colmajor(M, N, dtype)
    C0 = C.clone()
    run_gemm(A, B, C, ta, tb, -1.0, 1.0)
    opA = (A.t() if ta else A).double()
    opB = (B.t() if tb else B).double()
    ref = C0.double() - opA @ opB
    err = (C.double() - ref).abs().max().item()
    scale = (opA.abs() @ opB.abs()).max().item()
    tol = 1e-13 if dtype == torch.float64 else 2e-3  # tf32 operands: 2^-11 relative per product
    assert err <= tol * scale, (err, scale)
