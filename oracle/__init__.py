"""CPU fp64 oracle for the Luffy token-condensed MoE layer -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import it.
The product path (paper_2411_15419_b200) never imports or calls anything here.
"""
from .luffy_oracle import *  # noqa: F401,F403
