"""TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's RNS-CKKS hot path, used as the parity
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg.  The product (paper_2310_16530_b200) never imports it.
Pinned against the unmodified reference via tests/golden/ (see
tests/test_oracle.py).
"""
