"""Alias of paper_2206_06079_b200.engine (test infrastructure, see __init__)."""
import sys

from paper_2206_06079_b200 import engine as _m

sys.modules[__name__] = _m
