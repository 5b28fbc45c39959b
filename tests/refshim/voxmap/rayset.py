"""Alias of paper_2206_06079_b200.rayset (test infrastructure, see __init__)."""
import sys

from paper_2206_06079_b200 import rayset as _m

sys.modules[__name__] = _m
