"""Shared helpers for the GPU parity tests (product executor vs the C oracle)."""
import numpy as np
import torch

from oracle import bd


def to_oracle_layout(k, flat_block: np.ndarray, model: str = "resnet") -> np.ndarray:
    """Product block params (padded input channels for block 0: 16 bf16 / 32 fp32) -> oracle flat layout."""
    from paper_2301_12443_b200.executor import student_layout, stored_channels
    lay, _ = student_layout(k, model)
    g = bd.geom(k)
    cin, cout = g["cin"], g["cout"]
    mid = cout // 2
    cs = stored_channels(cin, model)
    parts = []
    for name in ("w1", "w2", "wsc", "g1", "b1", "g2", "b2", "gsc", "bsc"):
        o, n = lay[name]
        v = flat_block[o:o + n]
        if name == "w1":
            v = v.reshape(mid, 3, 3, cs)[..., :cin].reshape(-1)
        elif name == "wsc":
            v = v.reshape(cout, 1, 1, cs)[..., :cin].reshape(-1)
        parts.append(v)
    return np.concatenate(parts)


def partition_params(part, k) -> np.ndarray:
    base, _, total = part.layouts[k]
    flat = part.params()[base:base + total].cpu().numpy()
    return to_oracle_layout(k, flat, part.model)


def bf16_to_np(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


def compare_bf16_tensors(got: np.ndarray, want: np.ndarray, depth=1):
    """Both bf16-valued. After one bf16-rounded layer most elements are bit-identical and
    the rest one bf16 ulp apart (fp32 accumulation order differs); the differences compound
    with the number of stacked layers `depth`, so the bounds scale with it:
      max |diff|  <= depth * 2^-7 * max|want|      (a bf16 ulp per layer at full scale)
      mean |diff| <= depth * 2^-11 * max|want|."""
    assert got.shape == want.shape, (got.shape, want.shape)
    diff = np.abs(got.astype(np.float64) - want.astype(np.float64))
    scale = float(np.abs(want).max()) + 1e-12
    stats = dict(mismatch=float(np.mean(diff > 0)), max=float(diff.max() / scale), mean=float(diff.mean() / scale))
    assert stats["max"] <= depth * 2 ** -7, stats
    assert stats["mean"] <= depth * 2 ** -11, stats
    if depth == 1:
        assert stats["mismatch"] <= 0.05, stats
    return stats


def pad_image(x: np.ndarray) -> np.ndarray:
    """[n,32,32,3] -> [n,32,32,16] zero padded (the product's stored image layout)."""
    out = np.zeros(x.shape[:3] + (16,), np.float32)
    out[..., :3] = x
    return out
