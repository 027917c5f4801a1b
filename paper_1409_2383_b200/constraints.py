"""Constraint specifications of the drop-in API (reference constraints.py:27-69).

The B200 path implements the non-negative projection (constraints.py:105-111),
fused into the per-mode update kernel; row-stochastic rows (equality-
constrained solve + simplex projection) likewise; the global cardinality
projection (constraints.py:95-102) runs as a select + apply kernel pair
after the last-sweep update.  The cardinality constraint
needs the whole factor on one GPU, so the sharded path rejects it.
"""

from __future__ import annotations

from dataclasses import dataclass

_KINDS = ("nonneg", "nonneg_card", "row_stochastic")


@dataclass(frozen=True)
class ConstraintSpec:
    kind: str
    card: int | None = None

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown constraint kind {self.kind!r}")
        if self.kind == "nonneg_card":
            if self.card is None or int(self.card) < 1:
                raise ValueError("nonneg_card requires a positive nonzero budget")
            object.__setattr__(self, "card", int(self.card))
        elif self.card is not None:
            raise ValueError(f"{self.kind} takes no cardinality parameter")

    @classmethod
    def nonneg(cls) -> "ConstraintSpec":
        return cls("nonneg")

    @classmethod
    def nonneg_card(cls, c: int) -> "ConstraintSpec":
        return cls("nonneg_card", c)

    @classmethod
    def row_stochastic(cls) -> "ConstraintSpec":
        return cls("row_stochastic")

    @classmethod
    def parse(cls, name: str) -> "ConstraintSpec":
        name = name.strip()
        if name in ("nonneg", "row_stochastic"):
            return cls(name)
        if name.startswith("nonneg_card:"):
            return cls.nonneg_card(int(name.split(":", 1)[1]))
        raise ValueError(f"unknown constraint name {name!r}")

    def name(self) -> str:
        return f"nonneg_card:{self.card}" if self.kind == "nonneg_card" else self.kind


def normalize_specs(specs, order: int) -> list[ConstraintSpec]:
    """solver.normalize_specs (reference solver.py:154-164)."""
    if specs is None:
        specs = ConstraintSpec.nonneg()
    if isinstance(specs, ConstraintSpec):
        specs = [specs] * order
    else:
        specs = list(specs)
        if len(specs) != order:
            raise ValueError(f"need one constraint per mode ({order}), got {len(specs)}")
    for s in specs:
        if getattr(s, "kind", None) not in _KINDS:
            raise ValueError(f"unknown constraint {s!r}")
    return specs


# plan codes (include/ntf_b200.h: ntf_constraint)
_CODES = {"nonneg": 0, "nonneg_card": 1, "row_stochastic": 2}


def plan_codes(specs, dims, rank: int) -> tuple[list[int], list[int]]:
    """Per-mode (constraint code, cardinality budget) for the plan descriptor,
    with the reference's budget check (solver.py:359-363)."""
    codes, cards = [], []
    for d, s in zip(dims, specs):
        if s.kind == "nonneg_card" and s.card > d * rank:
            raise ValueError(f"cardinality budget {s.card} exceeds factor size {d}x{rank}")
        codes.append(_CODES[s.kind])
        cards.append(int(s.card) if s.kind == "nonneg_card" else 0)
    return codes, cards
