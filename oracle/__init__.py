"""CPU oracle for the ASADMM iteration loop -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  See oracle/admm_ref.py for the restatement and its
reference citations.
"""
