"""ORACLE — test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline — never as the product path.  The product (paper_2208_14049_b200)
never imports it.

Two layers:
  * ``restate`` — a plain-Python/numpy restatement of the reference's placement,
    search, cost model and combination fold, each function citing the
    reference file:line it follows;
  * ``refcpu`` — ctypes over oracle/_ref/libenserve_ref.so (the UNMODIFIED
    reference compiled from /root/reference by oracle/Makefile, with the oracle
    CPU member behind its PredictorFactory) and over liboracle.so (the CPU
    member restatement, cpu_member.c).
"""
