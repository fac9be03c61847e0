"""Seeded Balding-Nichols genotype specs for the BASELINE.json configs
(product side). The specs live in `workloads.py` (pure numpy, no libgkb);
this module adds the GklOptions of each config.
"""
from __future__ import annotations

from .gkl import GklOptions, ReorthMode, RestartMode
from .workloads import (CONFIG_OPTIONS, CONFIG_TEXT, OPTIONS_TEXT, SynthSpec,  # noqa: F401
                        balding_nichols, config_spec)


def config_options(cfg: int) -> GklOptions:
    """GklOptions per SURVEY.md 8d (workloads.CONFIG_OPTIONS)."""
    if cfg not in CONFIG_OPTIONS:
        raise ValueError(f"unknown config {cfg}")
    d = dict(CONFIG_OPTIONS[cfg])
    d["reorth"] = ReorthMode(d["reorth"])
    d["restart"] = RestartMode(d["restart"])
    return GklOptions(**d)
