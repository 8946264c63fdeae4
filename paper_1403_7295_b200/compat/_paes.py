"""`import _paes` for callers of the reference's Python module.

Put this directory on the module path (PYTHONPATH=<repo>/paper_1403_7295_b200/compat)
and code written against the reference's pybind11 module
(proj/python/paes_module.cpp) imports the B200 engine under the same name:
same functions, arguments, defaults for the strategies it knows, and
exceptions (see paper_1403_7295_b200/paes.py).
"""
import os as _os
import sys as _sys

_root = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
if _root not in _sys.path:
    _sys.path.insert(0, _root)

from paper_1403_7295_b200.paes import *  # noqa: E402,F401,F403
from paper_1403_7295_b200.paes import GpuError, IoError, PaddingError, WorkerError  # noqa: E402,F401
