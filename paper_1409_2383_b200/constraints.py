"""Constraint specifications of the drop-in API (reference constraints.py:27-69).

The B200 path implements the non-negative projection (constraints.py:105-111),
fused into the per-mode update kernel.  The cardinality and row-stochastic
kinds are accepted by ``ConstraintSpec`` for API compatibility but ``fit``
raises NotImplementedError for them.
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
    """solver.normalize_specs (reference solver.py:154-164), plus the B200
    envelope check (nonneg only)."""
    if specs is None:
        specs = ConstraintSpec.nonneg()
    if isinstance(specs, ConstraintSpec):
        specs = [specs] * order
    else:
        specs = list(specs)
        if len(specs) != order:
            raise ValueError(f"need one constraint per mode ({order}), got {len(specs)}")
    for s in specs:
        if getattr(s, "kind", None) != "nonneg":
            raise NotImplementedError(
                f"constraint {getattr(s, 'kind', s)!r} is outside the B200 path (nonneg only)")
    return specs
