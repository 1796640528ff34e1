"""Experiment: cap the rows of a direct chunk (default 256) for c3's sparse mode."""
import os, runpy, sys
sys.path.insert(0, os.getcwd())
import paper_2309_09131_b200._lib as lib
cap = int(os.environ["DIRECT_CAP"])
real_load = lib.load
class Proxy:
    def __init__(self, L): self.L = L
    def __getattr__(self, n):
        f = getattr(self.L, n)
        if n == "fc_chunk_rows_max":
            return lambda nm, r, m: min(f(nm, r, m), max(m, cap // m * m))
        return f
def load():
    return Proxy(real_load())
import paper_2309_09131_b200.layout as layout
layout._lib.load = load
sys.argv = ["bench.py", "--config", "3", "--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
runpy.run_path("bench.py", run_name="__main__")
