"""float64 CPU oracle for the rdFFT hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package.  It shares no code with paper_2511_01385_b200.
"""
from .rdfft_oracle import *  # noqa: F401,F403
