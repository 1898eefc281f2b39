"""Chance-constrained GP-MPPI planner for skid-steer robots.

Drop-in for the reference's Python package `gpmppi` (python/gpmppi/__init__.py, which
re-exports the pybind11 module `_gpmppi`, bindings/module.cpp:36-219): the same names
re-exported from paper_2411_03289_b200.pymodule, backed by the B200 library.
"""
from paper_2411_03289_b200.pymodule import *  # noqa: F401,F403
from paper_2411_03289_b200.pymodule import __doc__ as _doc

__doc__ = _doc
__version__ = "0.1.0"
