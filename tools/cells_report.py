"""Executed 1F1B cells per candidate for configs 2-4 (HSIM_LIB selects a variant)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hsim_inputs as H  # noqa: E402
from paper_2508_05370_b200 import Sim  # noqa: E402

for c in [int(x) for x in sys.argv[1:]] or [2, 3, 4]:
    s = Sim(H.get(c))
    n = s.space_size()
    print(os.path.basename(os.environ.get("HSIM_LIB", "default")), c, n, round(s.count_cells(0, n) / n, 1), flush=True)
