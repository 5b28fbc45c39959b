"""Alias of paper_2206_06079_b200.exporters (test infrastructure, see __init__)."""
import sys

from paper_2206_06079_b200 import exporters as _m

sys.modules[__name__] = _m
