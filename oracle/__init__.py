"""CPU oracle for the vmfilt hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  It is the parity checker, never
the thing measured as the product or shipped in its path.
"""
