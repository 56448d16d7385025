"""Test infrastructure only: CPU restatement of the reference slab FFT.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product path
(paper_1406_5597_b200) never imports it.
"""
from .slabfft_oracle import *  # noqa: F401,F403
