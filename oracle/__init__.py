"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see lightbeam_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
"""
