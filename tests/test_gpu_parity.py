"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs (tolerances: north star -- max relative error
normalised by ||tril(ref)||_F <= 1e-10 fp64, <= 1e-4 fp32)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_1602_07527_b200 as cd
import synthetic
from gpu_helpers import fp32_round, nerr, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL64, TOL32 = 1e-10, 1e-4

SIZES = [1, 2, 3, 5, 8, 16, 31, 32, 33, 47, 63, 64, 65, 100, 127, 128, 129, 200, 255, 256, 257, 300, 517]


def oracle_rev(L, Lb):
    return np.stack([oracle.chol_rev(L[b], Lb[b]) for b in range(L.shape[0])]) if L.ndim == 3 else oracle.chol_rev(L, Lb)


def oracle_fwd(L, Sd):
    if L.ndim == 3:
        return np.stack([oracle.chol_fwd(L[b], np.tril(Sd[b])) for b in range(L.shape[0])])
    return oracle.chol_fwd(L, np.tril(Sd))


@pytest.mark.parametrize("n", SIZES)
def test_rev_single_f64(n):
    L, Lb, _ = synthetic.draw(n, n)
    out = cd.chol_rev(to_dev(L), to_dev(Lb))
    assert nerr(to_host(out), oracle.chol_rev(L, Lb)) < TOL64


@pytest.mark.parametrize("n", SIZES)
def test_fwd_single_f64(n):
    L, _, Sd = synthetic.draw(n, 1000 + n, sdot=True)
    out = cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd)))
    assert nerr(to_host(out), oracle_fwd(L, Sd)) < TOL64


@pytest.mark.parametrize("n,nb", [(300, 1), (300, 2), (300, 3), (300, 7), (300, 16), (300, 32), (300, 33),
                                  (300, 64), (300, 100), (300, 128), (129, 128), (160, 31)])
def test_nb_sweep(n, nb):
    # any partition; SPEC.md:301 nb-invariance
    L, Lb, Sd = synthetic.draw(n, 77, sdot=True)
    r = cd.chol_rev(to_dev(L), to_dev(Lb), nb=nb)
    assert nerr(to_host(r), oracle.chol_rev(L, Lb)) < TOL64
    f = cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd)), nb=nb)
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL64


def test_nb_too_large_is_unsupported():
    L, Lb, _ = synthetic.draw(300, 1)
    with pytest.raises(cd.CholdiffError):
        cd.chol_rev(to_dev(L), to_dev(Lb), nb=256)


@pytest.mark.parametrize("n", [17, 32, 64, 200, 300])
@pytest.mark.parametrize("pad", [1, 2, 3])
def test_leading_dimension(n, pad):
    # odd ld -> cp.async GEMM / reg32 fallbacks; even ld -> TMA / left-looking / bulk32 paths with ld > n
    L, Lb, Sd = synthetic.draw(n, 5 * n + pad, sdot=True)
    Ld, Ad = to_dev(L, ld_pad=pad), to_dev(Lb, ld_pad=pad)
    assert Ld.stride(-1) == n + pad
    out = cd.chol_rev(Ld, Ad)
    assert out.data_ptr() == Ad.data_ptr()  # in place
    assert nerr(to_host(out), oracle.chol_rev(L, Lb)) < TOL64
    f = cd.chol_fwd(to_dev(L, ld_pad=pad), to_dev(np.tril(Sd), ld_pad=pad))
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL64


@pytest.mark.parametrize("n", [1, 5, 8, 16, 17, 24, 32, 33, 64, 100, 128, 150, 300])
def test_strided_batched(n):
    B = 37 if n <= 128 else (5 if n < 300 else 3)
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=3 * n, sdot=True)
    r = cd.chol_rev(to_dev(L), to_dev(Lb))
    assert nerr(to_host(r), oracle_rev(L, Lb)) < TOL64
    f = cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd)))
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL64


@pytest.mark.parametrize("n", [9, 32, 96, 140])
def test_pointer_array_batched(n):
    B = 6
    L, Lb, _ = synthetic.draw_batch(n, B, seed=n)
    Ls = [to_dev(L[b]) for b in range(B)]
    As = [to_dev(Lb[b]) for b in range(B)]
    lp = torch.tensor([t.data_ptr() for t in Ls], dtype=torch.int64, device="cuda")
    ap = torch.tensor([t.data_ptr() for t in As], dtype=torch.int64, device="cuda")
    nbytes = cd.workspace_size("rev", torch.float64, n, B)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
    rc = cd.lib().cd_chol_rev_batched(0, n, lp.data_ptr(), n, ap.data_ptr(), n, B, None, ws.data_ptr(), nbytes,
                                      None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    out = np.stack([to_host(a) for a in As])
    assert nerr(out, oracle_rev(L, Lb)) < TOL64


@pytest.mark.parametrize("n,dt", [(9, 0), (32, 0), (96, 0), (140, 0), (300, 0), (64, 1), (200, 1)])
def test_pointer_array_batched_fwd(n, dt):
    # cd_chol_fwd_batched: device array of device pointers
    B = 5
    tdt = torch.float64 if dt == 0 else torch.float32
    L, _, Sd = synthetic.draw_batch(n, B, seed=7 * n + dt, lbar=False, sdot=True)
    if dt == 1:
        L, Sd = fp32_round(L, Sd)
    Ls = [to_dev(L[b], tdt) for b in range(B)]
    Fs = [to_dev(np.tril(Sd[b]), tdt) for b in range(B)]
    lp = torch.tensor([t.data_ptr() for t in Ls], dtype=torch.int64, device="cuda")
    fp = torch.tensor([t.data_ptr() for t in Fs], dtype=torch.int64, device="cuda")
    nbytes = cd.workspace_size("fwd", tdt, n, B)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
    info = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    rc = cd.lib().cd_chol_fwd_batched(dt, n, lp.data_ptr(), n, fp.data_ptr(), n, B, None, ws.data_ptr(), nbytes,
                                      info.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    assert not info.cpu().any()
    out = np.stack([to_host(f) for f in Fs])
    assert nerr(out, oracle_fwd(L, Sd)) < (TOL64 if dt == 0 else TOL32)


def test_inplace_non_colmajor_sensitivity_is_updated():
    # a row-major (ordinary contiguous) sensitivity is processed in a column-major copy
    # and the result copied back, so the in-place contract holds for every layout
    n = 150
    L, Lb, Sd = synthetic.draw(n, 12, sdot=True)
    Lt = to_dev(L)
    A_rm = torch.from_numpy(np.ascontiguousarray(Lb)).cuda()  # logical orientation, row-major memory
    r = cd.chol_rev(Lt, A_rm)
    assert r.data_ptr() == A_rm.data_ptr()
    assert nerr(to_host(A_rm), oracle.chol_rev(L, Lb)) < TOL64
    F_rm = torch.from_numpy(np.ascontiguousarray(np.tril(Sd))).cuda()
    f = cd.chol_fwd(Lt, F_rm)
    assert f.data_ptr() == F_rm.data_ptr()
    assert nerr(to_host(F_rm), oracle_fwd(L, Sd)) < TOL64
    keep = torch.from_numpy(np.ascontiguousarray(Lb)).cuda()
    out = cd.chol_rev(Lt, keep, inplace=False)
    assert torch.equal(keep.cpu(), torch.from_numpy(Lb))  # untouched
    assert nerr(to_host(out), oracle.chol_rev(L, Lb)) < TOL64


def test_check_raises_singular_factor():
    n = 200
    L, Lb, _ = synthetic.draw_batch(n, 3, seed=3)
    L[1, 57, 57] = 0.0
    with pytest.raises(cd.SingularFactorError) as e:
        cd.chol_rev(to_dev(L), to_dev(Lb), check=True)
    assert e.value.info == [0, 58, 0]
    with pytest.raises(cd.SingularFactorError):
        cd.chol_fwd(to_dev(L), to_dev(Lb), check=True)
    L[1, 57, 57] = 1.5
    cd.chol_rev(to_dev(L), to_dev(Lb), check=True)  # no error


@pytest.mark.parametrize("n,op", [(129, "rev"), (129, "fwd"), (130, "fused")])
def test_batch_above_grid_limit(n, op):
    # batches above 65535 on the paths whose kernels index matrices by gridDim.y/z
    # (blocked GEMMs, block inverses, the fused factorisation) run in chunks; spot-check matrices
    # in the first, second and third chunk against the oracle
    B = 65536 + 37
    L1, Lb1, Sd1 = synthetic.draw_batch(n, 4, seed=5, sdot=True)
    idx = np.arange(B) % 4
    picks = [0, 32767, 32768, 65535, 65536, B - 1]
    if op == "fused":
        Sig = np.einsum("bij,bkj->bik", L1, L1)
        A = to_dev(Sig)[torch.from_numpy(idx).cuda()]
        Ad = to_dev(np.tril(Sd1))[torch.from_numpy(idx).cuda()]
        A, Ad = cd.colmajor(A), cd.colmajor(Ad)
        Lo, Fo = cd.chol_fwd_fused(A, Ad)
        for b in picks:
            Lref = oracle.chol(Sig[idx[b]])
            assert nerr(to_host(Lo[b]), Lref) < TOL64
            assert nerr(to_host(Fo[b]), oracle.chol_fwd(Lref, np.tril(Sd1[idx[b]]))) < TOL64
        return
    Ld = cd.colmajor(to_dev(L1)[torch.from_numpy(idx).cuda()])
    if op == "rev":
        A = cd.colmajor(to_dev(Lb1)[torch.from_numpy(idx).cuda()])
        out = cd.chol_rev(Ld, A)
        refs = [oracle.chol_rev(L1[k], Lb1[k]) for k in range(4)]
    else:
        A = cd.colmajor(to_dev(np.tril(Sd1))[torch.from_numpy(idx).cuda()])
        out = cd.chol_fwd(Ld, A)
        refs = [oracle.chol_fwd(L1[k], np.tril(Sd1[k])) for k in range(4)]
    for b in picks:
        assert nerr(to_host(out[b]), refs[idx[b]]) < TOL64


@pytest.mark.parametrize("n", [1, 7, 32, 33, 100, 128, 200, 512])
def test_f32_vs_oracle_on_rounded_inputs(n):
    B = 4
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=11 * n, sdot=True)
    L, Lb, Sd = fp32_round(L, Lb, Sd)
    r = cd.chol_rev(to_dev(L, torch.float32), to_dev(Lb, torch.float32))
    assert nerr(to_host(r), oracle_rev(L, Lb)) < TOL32
    f = cd.chol_fwd(to_dev(L, torch.float32), to_dev(np.tril(Sd), torch.float32))
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL32


@pytest.mark.parametrize("n", [6, 32, 90, 260])
def test_out_modes(n):
    L, Lb, _ = synthetic.draw(n, 400 + n)
    sym = oracle.chol_rev_symbolic_sym(L, Lb)  # Eq. 9
    o_sym = to_host(cd.chol_rev(to_dev(L), to_dev(Lb), out="sym"))
    assert np.array_equal(o_sym, o_sym.T)
    assert np.abs(o_sym - sym).max() / np.linalg.norm(sym) < TOL64
    G = 0.5 * (sym + np.diag(np.diag(sym)))  # G = (S + S^T)/2: Eq. 9 with off-diagonals halved
    o_g = to_host(cd.chol_rev(to_dev(L), to_dev(Lb), out="grad"))
    assert np.array_equal(o_g, o_g.T)
    assert np.abs(o_g - G).max() / np.linalg.norm(G) < TOL64


@pytest.mark.parametrize("n", [5, 32, 70, 300])
def test_upper_triangle_never_read_nor_written(n):
    L, Lb, Sd = synthetic.draw(n, 9 + n, sdot=True)
    Lp, Ap = synthetic.poison_upper(L), synthetic.poison_upper(Lb)
    out = to_host(cd.chol_rev(to_dev(Lp), to_dev(Ap)))
    iu = np.triu_indices(n, 1)
    assert np.all(np.isnan(out[iu]))
    assert nerr(out, oracle.chol_rev(L, Lb)) < TOL64
    f = to_host(cd.chol_fwd(to_dev(Lp), to_dev(synthetic.poison_upper(np.tril(Sd)))))
    assert np.all(np.isnan(f[iu]))
    assert nerr(f, oracle_fwd(L, Sd)) < TOL64


@pytest.mark.parametrize("n", [4, 32, 64, 300])
def test_info_reports_singular_factor(n):
    B = 3
    L, Lb, _ = synthetic.draw_batch(n, B, seed=1)
    L[1, n // 2, n // 2] = 0.0
    _, info = cd.chol_rev(to_dev(L), to_dev(Lb), info=True)
    assert info.cpu().tolist() == [0, n // 2 + 1, 0]
    _, info = cd.chol_fwd(to_dev(L), to_dev(np.tril(Lb)), info=True)
    assert info.cpu().tolist() == [0, n // 2 + 1, 0]


def test_zero_sizes():
    e = torch.empty(0, 0, dtype=torch.float64, device="cuda")
    cd.chol_rev(e, e.clone())
    eb = torch.empty(0, 4, 4, dtype=torch.float64, device="cuda")
    cd.chol_rev(eb, eb.clone())


@pytest.mark.parametrize("n", [32, 64, 300])
def test_power_of_two_scaling_bit_exact(n):
    # property holding at any size for a deterministic kernel
    L, Lb, _ = synthetic.draw(n, 123)
    a = to_host(cd.chol_rev(to_dev(L), to_dev(Lb)))
    b = to_host(cd.chol_rev(to_dev(L * 4.0), to_dev(Lb)))
    c = to_host(cd.chol_rev(to_dev(L), to_dev(Lb * 0.125)))
    assert np.array_equal(np.tril(b), np.tril(a) * 0.25)
    assert np.array_equal(np.tril(c), np.tril(a) * 0.125)


def test_deterministic():
    L, Lb, _ = synthetic.draw(700, 3)
    a = to_host(cd.chol_rev(to_dev(L), to_dev(Lb)))
    b = to_host(cd.chol_rev(to_dev(L), to_dev(Lb)))
    assert np.array_equal(np.tril(a), np.tril(b))


@pytest.mark.parametrize("n", [200, 300, 301, 1024])
def test_host_buffer_path(n):
    # even n: the pipelined copies (lower part of each column block streamed in / out);
    # odd n: dense copies.  Upper triangles are NaN-poisoned and must come back untouched.
    L, Lb, Sd = synthetic.draw(n, 8 + n, sdot=True)

    def host(m):
        return torch.from_numpy(synthetic.to_colmajor(synthetic.poison_upper(m))).transpose(0, 1).pin_memory()

    iu = np.triu_indices(n, 1)
    Lh, Ah = host(L), host(Lb)
    cd.chol_host("rev", Lh, Ah)
    out = Ah.numpy()
    assert nerr(out, oracle.chol_rev(L, Lb)) < TOL64
    assert np.all(np.isnan(out[iu]))
    h2d, d2h = cd.host_bytes()
    assert 0 < d2h <= n * n * 8 and h2d > 0
    if n >= 1024:  # pipelined: lower triangles (+ the diagonal blocks once more) only
        assert h2d < 0.7 * 2 * n * n * 8 and d2h < 0.7 * n * n * 8
    Fh = host(np.tril(Sd))
    cd.chol_host("fwd", host(L), Fh)
    f = Fh.numpy()
    assert nerr(f, oracle_fwd(L, Sd)) < TOL64
    assert np.all(np.isnan(f[iu]))


@pytest.mark.parametrize("n", [1, 5, 8, 17, 32, 33, 64])
def test_symbolic_route(n):
    # north star (d) / PAPER.md:748-754: Eq. 10 (reverse) and Eq. 8 (forward) on the whole matrix
    B = 5
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=70 + n, sdot=True)
    r = cd.chol_rev(to_dev(L), to_dev(Lb), route="symbolic")
    assert nerr(to_host(r), oracle_rev(L, Lb)) < TOL64
    f = cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd)), route="symbolic")
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL64
    for mode in ("sym", "grad"):  # output conventions through the same store
        a = to_host(cd.chol_rev(to_dev(L), to_dev(Lb), route="symbolic", out=mode))
        b = to_host(cd.chol_rev(to_dev(L), to_dev(Lb), out=mode))
        assert np.abs(a - b).max() / np.linalg.norm(b.reshape(B, -1), axis=1).min() < TOL64
    # fp32 on the rounded inputs
    L32, Lb32 = fp32_round(L, Lb)
    r32 = cd.chol_rev(to_dev(L32, torch.float32), to_dev(Lb32, torch.float32), route="symbolic")
    assert nerr(to_host(r32), oracle_rev(L32, Lb32)) < TOL32


def test_symbolic_route_upper_never_read_and_limits():
    n = 40
    L, Lb, _ = synthetic.draw(n, 4)
    out = to_host(cd.chol_rev(to_dev(synthetic.poison_upper(L)), to_dev(synthetic.poison_upper(Lb)),
                              route="symbolic"))
    assert np.all(np.isnan(out[np.triu_indices(n, 1)]))
    assert nerr(out, oracle.chol_rev(L, Lb)) < TOL64



@pytest.mark.parametrize("n", [1, 7, 64, 128, 129, 300, 517, 1024])
def test_chol_fwd_fused(n):
    # factorisation (oracle chol_unblocked PAPER.md:437-445)
    # and forward mode accumulated in one sweep
    B = 2 if n <= 300 or n == 1024 else 1
    L, _, Sd = synthetic.draw_batch(n, B, seed=900 + n, sdot=True)
    Sig = np.einsum("bij,bkj->bik", L, L)  # Sigma = L L^T
    Lref = np.stack([oracle.chol(Sig[b]) for b in range(B)])
    Fref = oracle_fwd(Lref, Sd)
    A = to_dev(synthetic.poison_upper(Sig) if B == 1 else Sig)
    Ad = to_dev(np.tril(Sd))
    Lo, Fo = cd.chol_fwd_fused(A, Ad)
    assert nerr(to_host(Lo), Lref) < TOL64
    assert nerr(to_host(Fo), Fref) < TOL64
    if B == 1:
        assert np.all(np.isnan(to_host(Lo)[0][np.triu_indices(n, 1)]))


def test_chol_fwd_fused_reports_indefinite():
    n = 300
    L, _, Sd = synthetic.draw(n, 5, sdot=True)
    Sig = L @ L.T
    Sig[200, 200] = -1.0  # not positive definite from pivot 201 on at the latest
    _, _, info = cd.chol_fwd_fused(to_dev(Sig), to_dev(np.tril(Sd)), info=True)
    assert 0 < int(info.cpu()[0]) <= 201


@pytest.mark.parametrize("n,B", [(1100, 1), (2048, 1), (300, 3)])
def test_f32_blocked_sizes(n, B):
    # fp32 blocked paths (tf32 tcgen05 GEMMs, fp64-arithmetic diagonal blocks) beyond the
    # batched configs: single large matrices with a ragged block and a batch of mid-size ones
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=31 + n, sdot=True)
    L, Lb, Sd = fp32_round(L, Lb, Sd)
    r = cd.chol_rev(to_dev(L, torch.float32), to_dev(Lb, torch.float32))
    assert nerr(to_host(r), oracle_rev(L, Lb)) < TOL32
    f = cd.chol_fwd(to_dev(L, torch.float32), to_dev(np.tril(Sd), torch.float32))
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL32


@pytest.mark.parametrize("n", [1024, 1100, 1537])
def test_f32_left_looking_nan_upper(n):
    # fp32 single matrices n >= 1024 take the left-looking tcgen05 schedule (k_symm_tc): the upper
    # triangles (NaN here) must never be read, ragged top-left block included
    L, Lb, _ = synthetic.draw(n, 61 + n)
    L, Lb = fp32_round(L, Lb)
    nan_up = np.triu(np.full((n, n), np.nan), 1)
    r = cd.chol_rev(to_dev(L + nan_up, torch.float32), to_dev(Lb + nan_up, torch.float32))
    out = to_host(r)
    assert np.all(np.isnan(np.triu(out, 1)[np.triu_indices(n, 1)]))  # upper never written
    assert nerr(out, oracle.chol_rev(L, Lb)) < 2.5e-5


@pytest.mark.parametrize("n,B,dt", [(300, 3, torch.float64), (512, 2, torch.float32), (40, 5, torch.float64),
                                    (1100, 1, torch.float32), (700, 1, torch.float64)])
def test_rev_fwd_two_streams_equal_separate_calls(n, B, dt):
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=8 * n, sdot=True)
    Lt, Lbt, St = to_dev(L, dt), to_dev(Lb, dt), to_dev(np.tril(Sd), dt)
    r1 = cd.chol_rev(Lt, Lbt.clone())
    f1 = cd.chol_fwd(Lt, St.clone())
    r2, f2 = cd.chol_rev_fwd(Lt, Lbt.clone(), St.clone())
    torch.cuda.synchronize()
    assert torch.equal(torch.tril(r1), torch.tril(r2)) and torch.equal(torch.tril(f1), torch.tril(f2))


@pytest.mark.parametrize("nb", [64, 128])
def test_f32_tf32_rounded_operands(nb):
    # the tcgen05 GEMM rounds its operands to tf32 (cvt.rna) instead of letting the
    # MMA truncate them: config-4-shaped matrices (n = 512) land near 1e-5 (truncation: 4.3e-5)
    L, Lb, Sd = synthetic.draw_batch(512, 4, seed=543, sdot=True)
    L, Lb, Sd = fp32_round(L, Lb, Sd)
    r = cd.chol_rev(to_dev(L, torch.float32), to_dev(Lb, torch.float32), nb=nb)
    assert nerr(to_host(r), np.stack([oracle.chol_rev(L[b], Lb[b]) for b in range(4)])) < 2.5e-5
    f = cd.chol_fwd(to_dev(L, torch.float32), to_dev(np.tril(Sd), torch.float32), nb=nb)
    assert nerr(to_host(f), np.stack([oracle.chol_fwd(L[b], Sd[b]) for b in range(4)])) < 2.5e-5


@pytest.mark.parametrize("n", [2048, 2500])
def test_f64_blocked_larger(n):
    # several hundred stream-K pieces and panel steps, ragged last block (2500), fused paths
    L, Lb, Sd = synthetic.draw(n, 55 + n, sdot=True)
    r = cd.chol_rev(to_dev(L), to_dev(Lb))
    assert nerr(to_host(r), oracle.chol_rev(L, Lb)) < TOL64
    f = cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd)))
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL64


def _guarded(m: np.ndarray, dtype, pad: int, gap: int):
    """Column-major device copy of (B, n, n) `m` inside a larger buffer: `pad` guard rows below
    each column (ld = n + pad) and `gap` guard columns between matrices (batch stride
    (n + gap) * ld), all guard cells NaN.  Returns (view, underlying buffer, guard mask)."""
    B, n = m.shape[0], m.shape[-1]
    ld = n + pad
    buf = np.full((B, n + gap, ld), np.nan)  # [b][column][row]
    buf[:, :n, :n] = np.swapaxes(m, -1, -2)
    guard = np.ones_like(buf, dtype=bool)
    guard[:, :n, :n] = False
    t = torch.from_numpy(buf).to(dtype).cuda()
    view = t[:, :n, :n].transpose(-1, -2)  # logical (B, n, n), strides (ld*(n+gap), 1, ld)
    return view, t, guard


@pytest.mark.parametrize("n,B,dt", [(32, 9, torch.float64), (24, 5, torch.float64), (64, 4, torch.float64),
                                    (300, 2, torch.float64), (129, 2, torch.float64), (300, 2, torch.float32),
                                    (512, 2, torch.float32)])
def test_no_writes_outside_the_matrices(n, B, dt):
    # every path writes only inside tril of its matrices: NaN guard rows (ld > n) and guard
    # columns between batch entries (stride > n * ld) must come back untouched
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=3 + n, sdot=True)
    if dt == torch.float32:
        L, Lb, Sd = fp32_round(L, Lb, Sd)
    for op, src, ref in (("rev", Lb, oracle_rev(L, Lb)), ("fwd", np.tril(Sd), oracle_fwd(L, Sd))):
        Lv, _, _ = _guarded(L, dt, 2, 3)
        Av, Abuf, guard = _guarded(src, dt, 2, 3)
        out = cd.chol_rev(Lv, Av) if op == "rev" else cd.chol_fwd(Lv, Av)
        assert out.data_ptr() == Av.data_ptr()
        assert nerr(to_host(out), ref) < (TOL64 if dt == torch.float64 else TOL32)
        assert np.all(np.isnan(to_host(Abuf)[guard]))


@pytest.mark.parametrize("n,B", [(40, 3), (300, 2)])
def test_no_writes_outside_symbolic_and_fused(n, B):
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=8 + n, sdot=True)
    if n <= 64:
        Lv, _, _ = _guarded(L, torch.float64, 2, 3)
        Av, Abuf, guard = _guarded(Lb, torch.float64, 2, 3)
        out = cd.chol_rev(Lv, Av, route="symbolic")
        assert nerr(to_host(out), oracle_rev(L, Lb)) < TOL64
        assert np.all(np.isnan(to_host(Abuf)[guard]))
    S = np.einsum("bij,bkj->bik", L, L)
    Sv, Sbuf, g1 = _guarded(S, torch.float64, 2, 3)
    Dv, Dbuf, g2 = _guarded(np.tril(Sd), torch.float64, 2, 3)
    Lo, Fo = cd.chol_fwd_fused(Sv, Dv)
    Lref = np.stack([oracle.chol(S[b]) for b in range(B)])
    assert nerr(to_host(Lo), Lref) < TOL64
    assert nerr(to_host(Fo), oracle_fwd(Lref, Sd)) < TOL64
    assert np.all(np.isnan(to_host(Sbuf)[g1])) and np.all(np.isnan(to_host(Dbuf)[g2]))


@pytest.mark.parametrize("n,B", [(65, 3), (200, 2), (300, 1), (517, 1)])
def test_symbolic_route_large(n, B):
    # Eqs. 10 / 8 on the whole matrix via blocked triangular solves
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=600 + n, sdot=True)
    r = cd.chol_rev(to_dev(L), to_dev(Lb), route="symbolic")
    assert nerr(to_host(r), oracle_rev(L, Lb)) < TOL64
    f = cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd)), route="symbolic")
    assert nerr(to_host(f), oracle_fwd(L, Sd)) < TOL64
    g = to_host(cd.chol_rev(to_dev(L), to_dev(Lb), route="symbolic", out="grad"))
    g0 = to_host(cd.chol_rev(to_dev(L), to_dev(Lb), out="grad"))
    assert np.abs(g - g0).max() / np.linalg.norm(g0.reshape(B, -1), axis=1).min() < TOL64
    L32, Lb32, Sd32 = fp32_round(L, Lb, Sd)
    r32 = cd.chol_rev(to_dev(L32, torch.float32), to_dev(Lb32, torch.float32), route="symbolic")
    assert nerr(to_host(r32), oracle_rev(L32, Lb32)) < TOL32
    f32 = cd.chol_fwd(to_dev(L32, torch.float32), to_dev(np.tril(Sd32), torch.float32), route="symbolic")
    assert nerr(to_host(f32), oracle_fwd(L32, Sd32)) < TOL32


@pytest.mark.parametrize("n,B,dt", [(64, 1, torch.float64), (32, 37, torch.float64), (300, 1, torch.float64),
                                    (300, 2, torch.float32)])
def test_cuda_graph_capture_and_replay(n, B, dt):
    # the library enqueues only stream-ordered work (launches, memsets, event fork/join of its
    # own streams), so a call can be captured once into a CUDA graph and replayed
    L, Lb, _ = synthetic.draw_batch(n, B, seed=44 + n)
    if dt == torch.float32:
        L, Lb = fp32_round(L, Lb)
    Ld, A0 = to_dev(L, dt), to_dev(Lb, dt)
    A = A0.clone().transpose(-1, -2).contiguous().transpose(-1, -2)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cd.chol_rev(Ld, A)  # warm-up outside capture (library streams, kernel attributes)
    torch.cuda.current_stream().wait_stream(s)
    A.copy_(A0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cd.chol_rev(Ld, A)
    for _ in range(3):
        A.copy_(A0)
        g.replay()
    torch.cuda.synchronize()
    assert nerr(to_host(A), oracle_rev(L, Lb)) < (TOL64 if dt == torch.float64 else TOL32)


@pytest.mark.parametrize("n,B,dt", [(512, 4, torch.float32), (300, 2, torch.float64)])
def test_rev_fwd_cuda_graph_and_info(n, B, dt):
    # cd_chol_rev_fwd forks the forward sweep onto a library stream and joins it back: the call can
    # be captured into a CUDA graph; d_info carries the reverse sweep's status (a zero pivot)
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=91 + n, sdot=True)
    if dt == torch.float32:
        L, Lb, Sd = fp32_round(L, Lb, Sd)
    Ld, A0, F0 = to_dev(L, dt), to_dev(Lb, dt), to_dev(np.tril(Sd), dt)
    A, F = A0.clone(), F0.clone()
    cd.chol_rev_fwd(Ld, A, F)  # warm-up outside capture (library streams and events)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cd.chol_rev_fwd(Ld, A, F)
    for _ in range(2):
        A.copy_(A0)
        F.copy_(F0)
        g.replay()
    torch.cuda.synchronize()
    tol = TOL64 if dt == torch.float64 else 2.5e-5
    Ah, Fh = to_host(A), to_host(F)
    for b in range(B):
        assert nerr(Ah[b], oracle.chol_rev(L[b], Lb[b])) < tol
        assert nerr(Fh[b], oracle.chol_fwd(L[b], np.tril(Sd[b]))) < tol
    # d_info through the C ABI: a zero pivot in matrix 1 at 1-based index 5
    Lz = L.copy()
    Lz[1, 4, 4] = 0.0
    Lzd = to_dev(Lz, dt)
    A2, F2 = A0.clone(), F0.clone()
    info = torch.zeros(B, dtype=torch.int32, device="cuda")
    Lk = cd.lib()
    o = cd._opts(None, "auto", "tril")
    dtc = cd.CD_F64 if dt == torch.float64 else cd.CD_F32
    nbytes = int(Lk.cd_workspace_size_rev_fwd(dtc, n, B, ctypes.byref(o)))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
    rc = Lk.cd_chol_rev_fwd_strided_batched(dtc, n, Lzd.data_ptr(), n, n * n, A2.data_ptr(), n, n * n, F2.data_ptr(),
                                            n, n * n, B, ctypes.byref(o), ws.data_ptr(), nbytes,
                                            ctypes.c_void_p(info.data_ptr()),
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    got = info.cpu().tolist()
    assert got[1] == 5 and all(v == 0 for i, v in enumerate(got) if i != 1)
