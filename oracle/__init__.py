"""CPU oracle for arXiv 1703.01202's DVD-PFC Newton-Krylov-Schwarz step.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
See pfc_oracle.c for the per-function citations and DESIGN.md §3 for the pins.
"""
from .oracle import *  # noqa: F401,F403
