"""Alias of paper_2206_06079_b200.config (test infrastructure, see __init__)."""
import sys

from paper_2206_06079_b200 import config as _m

sys.modules[__name__] = _m
