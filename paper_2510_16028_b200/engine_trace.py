"""Trace record (engine.py:288-298)."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class Trace:
    tensors: list
    profile_id: str
    input_digests: dict
    weight_digests: dict

    def __len__(self):
        return len(self.tensors)
