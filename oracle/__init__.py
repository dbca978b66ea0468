"""ORACLE / TEST INFRASTRUCTURE — CPU checkers for the B200 hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference) may
import this package. The product (paper_2503_01890_b200) never does.
"""
