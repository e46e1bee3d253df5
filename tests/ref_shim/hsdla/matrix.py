"""Shim of `hsdla.matrix` (see the package docstring): this package's storage types and HSM1."""
from paper_1602_06589_b200.hsm1 import HSM1_MAGIC, read_hsm1, write_hsm1  # noqa: F401
from paper_1602_06589_b200.matrix import *  # noqa: F401,F403
