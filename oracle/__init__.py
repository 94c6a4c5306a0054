"""ORACLE — test infrastructure only (CPU restatements used as checkers).

Imported only by tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline leg.
The product package paper_2502_19913_b200 never imports it.
"""
