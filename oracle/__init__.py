"""CPU oracle for the DGSM build + query (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  See oracle/dgsm_oracle.c.
"""
