"""Test infrastructure: CPU restatement oracle (see forest_oracle.py header).

Importable only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs; never by the product package.
"""
