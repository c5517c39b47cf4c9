"""ORACLE — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

CPU restatement of the reference's hot path (`spheregrid`, /root/reference/pkg/src) used
only as the checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product package (paper_1908_07038_b200/) never imports it.

Pinning: every function here is checked against the golden fixtures in tests/golden/,
which were produced by running the unmodified reference in this container
(tests/golden/make_golden.py); tests/test_oracle.py holds those checks.
"""
