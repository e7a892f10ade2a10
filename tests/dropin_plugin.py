"""pytest plugin: ragsim's OWN test suite with the drop-in engine substituted.

Loaded with ``-p tests.dropin_plugin`` before the reference's test modules are collected:
``ragsim.simulator.SimulationEngine`` becomes ``DropInEngine`` — this package's
``TieredEngine`` (TieredKnowledgeTree + the native block pool in accounting mode, one
token per block so the pool's block accounting must equal the tree's token accounting
exactly).  Every ``ragsim.run`` / ``measure_throughput`` / CLI run in those tests then
goes through the drop-in, and every tier transition the reference tree makes is
replayed on the native allocator (any mismatch raises ``CacheError``).
"""

from __future__ import annotations

from paper_2404_12457_b200 import _ragsim  # noqa: F401  (puts ragsim on sys.path)
from paper_2404_12457_b200.cache import TieredEngine
from paper_2404_12457_b200.pool import accounting_pool

import ragsim.simulator as _sim  # noqa: E402

_CAP = 1 << 22  # blocks per tier (the tests' 10**9-token "unbounded" tiers never fill it)
STATS = {"engines": 0}


class DropInEngine(TieredEngine):
    def __init__(self, config, trace, sizes, stage_provider=None):
        pool = accounting_pool(max(1, min(int(config.gpu_capacity_tokens), _CAP)),
                               max(0, min(int(config.host_capacity_tokens), _CAP)), 1)
        super().__init__(config, trace, sizes, stage_provider=stage_provider, pool=pool)
        STATS["engines"] += 1


_sim.SimulationEngine = DropInEngine


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"drop-in engines constructed: {STATS['engines']}")
