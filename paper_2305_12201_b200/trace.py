"""Run traces in the reference's JSON-lines wire format (simworkers.py:88-155).

``IterationRecord`` keeps the reference's fields in the reference's order, so
a trace written here reads back with the reference's ``RunTrace.from_jsonl``.
Beyond the reference, a record can carry CUDA-measured times of the step
(``measured``: milliseconds from events on the stream, e.g. the whole step,
the select, the exchange) beside the modeled ``t_*`` seconds the controller
decides on (decisions never read measured time).  They are written
under a ``"measured"`` key only when asked for (``to_jsonl(measured=True)``),
which keeps the default output readable by the reference.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from typing import Iterator

import numpy as np

REQUIRED_TRACE_FIELDS = ("iter", "cf", "gain_min", "gain_c", "t_o", "t_compress",
                         "t_s", "t_iter", "tsys", "tcomp", "loss",
                         "floats_sent", "words_sent")


@dataclass
class IterationRecord:
    """One trace row; field order is the wire order (simworkers.py:88-108)."""

    iter: int
    cf: float
    gain_min: float
    gain_c: float
    t_o: float
    t_compress: float
    t_s: float
    t_iter: float
    tsys: float
    tcomp: float
    loss: float
    floats_sent: int
    words_sent: int
    choice: str
    theta_min: float
    measured: dict = field(default_factory=dict, compare=False)

    def to_dict(self, measured: bool = False) -> dict:
        d = asdict(self)
        m = d.pop("measured")
        if measured and m:
            d["measured"] = m
        return d


@dataclass
class RunTrace:
    """Per-iteration records of a run, JSON-lines serialisable (simworkers.py:116-155)."""

    records: list[IterationRecord] = field(default_factory=list)

    def append(self, record: IterationRecord) -> None:
        self.records.append(record)

    def __len__(self) -> int:
        return len(self.records)

    def __iter__(self) -> Iterator[IterationRecord]:
        return iter(self.records)

    def column(self, name: str) -> np.ndarray:
        return np.asarray([getattr(r, name) for r in self.records])

    def measured_column(self, name: str) -> np.ndarray:
        """A CUDA-measured time per record (NaN where it was not measured)."""
        return np.asarray([r.measured.get(name, float("nan")) for r in self.records], dtype=np.float64)

    def total(self, name: str):
        values = self.column(name)
        return values.sum().item() if len(values) else 0

    def to_jsonl(self, measured: bool = False) -> str:
        return "".join(json.dumps(r.to_dict(measured)) + "\n" for r in self.records)

    @classmethod
    def from_jsonl(cls, path) -> "RunTrace":
        records = []
        with open(path, "r", encoding="utf-8") as fh:
            for line in fh:
                line = line.strip()
                if not line:
                    continue
                row = json.loads(line)
                missing = [f for f in REQUIRED_TRACE_FIELDS if f not in row]
                if missing:
                    raise ValueError(f"trace record missing fields {missing}")
                records.append(IterationRecord(**row))
        return cls(records)
