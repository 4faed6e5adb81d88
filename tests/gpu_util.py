"""Helpers shared by the GPU tests: numpy (oracle side) <-> torch CUDA (kernel side) marshalling only."""
import numpy as np
import torch


def to_dev_bf16(a: np.ndarray, ld: int | None = None) -> torch.Tensor:
    """uint16 bf16 bits [r][c] -> CUDA bf16 tensor [r][c] whose row stride is ld (>= c, multiple of 8)."""
    r, c = a.shape
    ld = ((c + 7) // 8 * 8) if ld is None else ld
    buf = torch.zeros((r, ld), dtype=torch.int16)
    buf[:, :c] = torch.from_numpy(a.view(np.int16))
    return buf.cuda().view(torch.bfloat16)[:, :c]


def to_dev_f32(a: np.ndarray, ld: int | None = None) -> torch.Tensor:
    r, c = a.shape
    ld = ((c + 3) // 4 * 4) if ld is None else ld
    buf = torch.zeros((r, ld), dtype=torch.float32)
    buf[:, :c] = torch.from_numpy(a)
    return buf.cuda()[:, :c]


def u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def u16(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def u8(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.uint8)


def packed_np(P):
    return u16(P.values), u8(P.col_idx), u32(P.meta)
