"""ORACLE -- TEST INFRASTRUCTURE ONLY (see qgs_oracle.py).

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg; never by the product package.
"""
