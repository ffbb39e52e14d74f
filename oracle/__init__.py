"""CPU oracle for the Optimus bubble-scheduling search — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2408_03505_b200/) never does, and the two share no code.
"""
