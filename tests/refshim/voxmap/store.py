"""Alias of paper_2206_06079_b200.store (test infrastructure, see __init__)."""
import sys

from paper_2206_06079_b200 import store as _m

sys.modules[__name__] = _m
