"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
import numpy as np
import torch

import synthetic


def to_dev(m: np.ndarray, dtype=torch.float64, ld_pad: int = 0) -> torch.Tensor:
    """Logical numpy (N,N)/(B,N,N) -> CUDA tensor, logical orientation, column-major memory
    (optionally with leading dimension N + ld_pad)."""
    n = m.shape[-1]
    if ld_pad:
        shape = m.shape[:-2] + (n, n + ld_pad)
        buf = np.full(shape, 7.0)  # padding rows hold junk that must never be read
        buf[..., :n, :n] = np.swapaxes(m, -1, -2)
        t = torch.from_numpy(buf).to(dtype).cuda()
        return t[..., :n].transpose(-1, -2) if m.ndim == 2 else t[..., :n].transpose(-1, -2)
    return torch.from_numpy(synthetic.to_colmajor(m)).to(dtype).cuda().transpose(-1, -2)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().double().cpu().numpy()


def nerr(out: np.ndarray, ref: np.ndarray) -> float:
    """max over the lower triangle |out - ref| / ||tril(ref)||_F (per matrix, max over batch)."""
    out = np.tril(out)
    ref = np.tril(ref)
    if ref.ndim == 2:
        out, ref = out[None], ref[None]
    num = np.abs(out - ref).reshape(ref.shape[0], -1).max(axis=1)
    den = np.linalg.norm(ref.reshape(ref.shape[0], -1), axis=1)
    den[den == 0] = 1.0
    return float((num / den).max())


def fp32_round(*arrs):
    """fp32 runs are compared with the fp64 oracle on fp32-rounded inputs."""
    return [None if a is None else a.astype(np.float32).astype(np.float64) for a in arrs]
