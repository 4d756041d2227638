"""Test infrastructure: CPU restatement of the reference hot path (the checker).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline legs may
import this package.  The product (`paper_1903_08690_b200`) never does.
"""
