"""Alias of paper_2206_06079_b200.tsdf (test infrastructure, see __init__)."""
import sys

from paper_2206_06079_b200 import tsdf as _m

sys.modules[__name__] = _m
