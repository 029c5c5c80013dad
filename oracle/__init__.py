"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see moba_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this package.
"""
