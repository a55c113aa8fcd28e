"""ORACLE — test infrastructure only (CPU restatements of the reference's hot path).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package, and only as the checker or the timed CPU baseline.
The product package never imports it.  Each module's header says how it is pinned
to the reference (golden fixtures made by tools/make_golden.py from the reference
itself).
"""
