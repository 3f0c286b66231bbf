"""The consumer-side contract check of the path (mirrors backend.assemble,
vlmfp/backend.py:92-109): the expanded prompt's image spans must carry exactly
``visual_token_count(plan)`` placeholder ids."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from .errors import AssemblyError
from .tokenred import TokenReductionConfig, visual_token_count


@dataclass(frozen=True)
class AssembledSequence:
    ids: list[int]
    n_visual: int
    n_text: int


def assemble(seq, plan: Optional[object], tr_cfg: TokenReductionConfig) -> AssembledSequence:
    """Raise AssemblyError(expected, got) unless sum(span lengths) matches the plan."""
    got = sum(length for _, length in seq.image_spans)
    expected = 0 if plan is None else visual_token_count(plan, tr_cfg.patch_edge, tr_cfg.r)
    if got != expected:
        raise AssemblyError(expected=expected, got=got)
    return AssembledSequence(ids=list(seq.ids), n_visual=got, n_text=len(seq.ids) - got)


__all__ = ["AssembledSequence", "assemble"]
