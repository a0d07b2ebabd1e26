"""Measures the engine's FP64-pipe roofline probe (ssb_fp64_peak)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine
from paper_2308_03399_b200.api import _fp64_peak
e = Engine(0)
for _ in range(3):
    print("fp64 ops/s", _fp64_peak(e), flush=True)
