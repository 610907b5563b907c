"""Loader for the reference-generated golden fixtures (tests/golden/cases)."""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from types import SimpleNamespace

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES_DIR = GOLDEN / "cases"


@dataclass(frozen=True)
class Layout:
    unit_bits: int
    units_per_subseq: int
    subseqs_per_seq: int

    @property
    def subseq_bits(self) -> int:
        return self.unit_bits * self.units_per_subseq

    @property
    def seq_bits(self) -> int:
        return self.subseq_bits * self.subseqs_per_seq


class Case:
    """Duck-typed stream (units/layout/total_bits/...) plus expected outputs."""

    def __init__(self, path: Path):
        self.name = path.stem
        z = np.load(path)
        self.d = {k: z[k] for k in z.files}
        d = self.d
        self.layout = Layout(int(d["unit_bits"]), int(d["ups"]), int(d["sps"]))
        self.units = d["units"].astype(np.uint32)
        self.total_bits = int(d["total_bits"])
        self.symbol_count = int(d["symbol_count"])
        self.gap = d["gap"].astype(np.uint8) if int(d["has_gap"]) else None
        lens = d["lens"]
        codes = d["codes"]
        nz = np.nonzero(lens)[0]
        self.codebook = SimpleNamespace(
            kind="canonical" if int(d["kind"]) == 0 else "explicit",
            entries={int(s): (int(codes[s]), int(lens[s])) for s in nz},
            symbol_width=int(d["symbol_width"]),
            lengths=lens.astype(np.uint8),
        )
        self.symbols = d["symbols_in"].astype(np.uint16)

    def __getitem__(self, k):
        return self.d[k]

    def has(self, k) -> bool:
        return k in self.d

    @property
    def num_subseqs(self) -> int:
        return -(-self.total_bits // self.layout.subseq_bits)

    @property
    def num_seqs(self) -> int:
        return -(-self.num_subseqs // self.layout.subseqs_per_seq)

    @property
    def corrupt(self) -> bool:
        return not self.has("oracle_starts")

    def __repr__(self):
        return f"Case({self.name})"


def all_cases() -> list[Case]:
    return [Case(p) for p in sorted(CASES_DIR.glob("*.npz"))]


def case(name: str) -> Case:
    return Case(CASES_DIR / f"{name}.npz")


def digests() -> dict:
    return json.loads((GOLDEN / "digests.json").read_text())
