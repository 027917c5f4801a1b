"""Test-infrastructure oracle (CPU restatement of the reference NTF path).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by the product package.
"""
