"""TEST INFRASTRUCTURE ONLY: CPU restatements of the reference (results oracle).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
