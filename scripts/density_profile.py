"""Runs the device density checker once on GHZ10 + depolarizing (n = 10, the
evolver's maximum) for ncu: gpurun -- ncu ... python scripts/density_profile.py"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program
g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "density_exact.json")))
c = next(x for x in g["cases"] if x["name"] == "ghz10_depol")
e = Engine(0)
p = Program.from_text(c["circuit"], c["noise"])
t = time.perf_counter()
d = e.exact_creg_distribution(p)
print("entries", len(d), "seconds %.4f" % (time.perf_counter() - t))
