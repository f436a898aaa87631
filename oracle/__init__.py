"""ORACLE -- test infrastructure only (see oracle/oracle.py).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg; never from the product package.  Parity of this restatement is
pinned against tests/golden/ (produced by executing the reference).
"""
