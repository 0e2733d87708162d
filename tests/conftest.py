import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# The segmenter sends large segments to the tcgen05 kernels only when they hold
# at least LORA_TC_MIN_ROWS rows in total (a perf heuristic, default 256); the
# parity tests pin each kernel route by segment size alone, so they run with
# the heuristic off (test_tc_min_rows_heuristic checks the default itself).
os.environ.setdefault("LORA_TC_MIN_ROWS", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI CUDA library)")
    config.addinivalue_line("markers", "slow: long-running")
