"""CPU oracle for the PipeFusion hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import, call, link or execute anything here, and
only as the checker or the CPU baseline -- never as the product path.
"""
