"""pytest plugin: run the REFERENCE's own test suite against the B200 drop-in.

    tools/stage_reference_suite.sh      # once: reference tests -> baseline/_ref/tests
    PYTHONPATH=baseline/_ref:. python -m pytest baseline/_ref/tests \
        -p tools.conformance_plugin -q

Before test collection it calls paper_1803_00737_b200.integration.install(),
which rebinds the reference's hot-path names (the binding sites listed in
SURVEY.md 8(b)) to the sm_100a drop-in, including
the cluster worker's handle_task. Nothing here computes.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_00737_b200 import integration  # noqa: E402

_HANDLE = None


def pytest_configure(config):
    global _HANDLE
    _HANDLE = integration.install()


def pytest_terminal_summary(terminalreporter):
    routed = _HANDLE.routed if _HANDLE is not None else {}
    terminalreporter.write_line("B200 drop-in calls routed: " +
                                ", ".join(f"{k}={v}" for k, v in sorted(routed.items())))
