"""Oracle package — TEST INFRASTRUCTURE ONLY (see oracle/Makefile, oracle/kvx_oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package. The product package never does.
"""
