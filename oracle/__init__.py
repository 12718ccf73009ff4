"""CPU oracle for the guided-filter hot path -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs.  The product package never imports it.  See gf_oracle.py's header for
how parity is pinned (golden vectors from the real reference).
"""
