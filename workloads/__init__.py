"""Seeded synthetic input generators shared by the tests and bench.py.

This module holds NO part of the method's arithmetic (no K-TanH, no
thresholds, no tables).  It only builds inputs with the shapes, sizes and
value distributions of BASELINE.json's `configs` (the paper's own workloads
are GNMT/WMT16 activations, which are not available; these
synthetic tensors stand in for them -- see DESIGN.md "Input recipe").

Both the oracle side and the CUDA side consume the *same bytes*: inputs are
generated once (on the device, with a seeded torch.Generator) and the tests
copy them to the host for the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Config:
    key: str
    desc: str
    shape: tuple
    dtype: torch.dtype
    dist: str        # "all_bf16" | "normal" | "uniform"
    scale: float     # std for normal, half-width for uniform
    seed: int
    ops: tuple       # which library calls the config exercises

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    @property
    def elem_bytes(self) -> int:
        return torch.tensor([], dtype=self.dtype).element_size()


# BASELINE.json "configs", in order.
CONFIGS = {
    "c1_exhaustive_bf16": Config(
        "c1_exhaustive_bf16", "all 65,536 BF16 bit patterns, K-TanH", (65536,),
        torch.bfloat16, "all_bf16", 0.0, 1, ("ktanh_bf16",)),
    "c2_bf16_2p24": Config(
        "c2_bf16_2p24", "BF16 K-TanH, 2^24 elements ~ N(0, 2^2), RNE cast", (1 << 24,),
        torch.bfloat16, "normal", 2.0, 2, ("ktanh_bf16",)),
    "c3_f32_2p28": Config(
        "c3_f32_2p28", "FP32 K-TanH, 2^28 elements ~ U[-8, 8]", (1 << 28,),
        torch.float32, "uniform", 8.0, 3, ("ktanh_f32",)),
    "c4_lstm_gates": Config(
        "c4_lstm_gates", "LSTM gates [128, 50, 4x1024] BF16 ~ N(0, 1.5^2); "
        "K-TanH on g, K-Sigmoid on i, f, o", (128, 50, 4 * 1024),
        torch.bfloat16, "normal", 1.5, 4, ("klstm_gates_bf16",)),
    "c5_ffn_2p30": Config(
        "c5_ffn_2p30", "FFN activations [65536, 16384] BF16 ~ N(0, 1) per GPU; "
        "K-GELU and K-Swish", (65536, 16384),
        torch.bfloat16, "normal", 1.0, 5, ("kgelu_bf16", "kswish_bf16")),
}

LSTM_HIDDEN = 1024


def all_bf16_patterns(device="cpu") -> torch.Tensor:
    """Every BF16 bit pattern 0x0000..0xFFFF in order, as a bfloat16 tensor."""
    w = torch.arange(65536, dtype=torch.int32).to(torch.int16)   # two's-complement wrap
    return w.view(torch.bfloat16).to(device)


def make_input(cfg: Config | str, device="cuda", rank: int = 0, numel: int | None = None,
               seed: int | None = None) -> torch.Tensor:
    """Generate the config's input.  `numel` overrides the size (flat) for
    reduced-size parity cases; `rank` offsets the seed (config 5 uses
    seed 5 + rank, independent per-GPU shards)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.dist == "all_bf16":
        return all_bf16_patterns(device)
    shape = cfg.shape if numel is None else (numel,)
    g = torch.Generator(device=device)
    g.manual_seed((cfg.seed if seed is None else seed) + rank)
    if cfg.dist == "normal":
        v = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
        v.mul_(cfg.scale)
    elif cfg.dist == "uniform":
        v = torch.rand(shape, generator=g, device=device, dtype=torch.float32)
        v.mul_(2 * cfg.scale).sub_(cfg.scale)
    else:
        raise ValueError(cfg.dist)
    if cfg.dtype == torch.float32:
        return v
    return v.to(cfg.dtype)   # round-to-nearest-even cast (BASELINE.json configs[1])


def special_values_bf16() -> list:
    """Bit patterns of the format's corner cases: +-0, subnormals, +-inf, NaNs,
    +-max finite, min normal."""
    return [0x0000, 0x8000, 0x0001, 0x8001, 0x007F, 0x0080, 0x7F7F, 0xFF7F,
            0x7F80, 0xFF80, 0x7FC0, 0xFFC0, 0x7F81, 0xFFFF]


def special_values_f32() -> list:
    return [0x00000000, 0x80000000, 0x00000001, 0x80000001, 0x007FFFFF, 0x00800000,
            0x7F7FFFFF, 0xFF7FFFFF, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000,
            0x7F800001, 0xFFFFFFFF]
