"""CPU fp64 oracle for the FlowMoE block hot path — TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never by paper_2510_00207_b200.
"""
from .flowmoe_oracle import *  # noqa: F401,F403
