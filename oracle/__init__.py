"""CPU fp64 oracle for the RunLoRA hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product package never imports it.
"""
from .runlora_oracle import *  # noqa: F401,F403
