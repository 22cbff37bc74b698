"""ORACLE package -- TEST INFRASTRUCTURE ONLY (see oracle/chebyshevt.py header).

May be imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product path never imports it.
"""
