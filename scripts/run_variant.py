"""Run a repo script against a variant library (tune/<variant>/libpaes_cuda.so):
    python scripts/run_variant.py tune/<variant>/libpaes_cuda.so scripts/<script>.py [args...]
The variant replaces paper_1403_7295_b200/lib/libpaes_cuda.so for that process only."""
import os
import runpy
import sys

sys.path.insert(0, os.getcwd())
from paper_1403_7295_b200 import _native as N  # noqa: E402

lib = os.path.abspath(sys.argv[1])
N.lib_path = lambda: lib
script = sys.argv[2]
sys.argv = [script] + sys.argv[3:]
sys.path.insert(0, os.path.dirname(os.path.abspath(script)))
runpy.run_path(script, run_name="__main__")
