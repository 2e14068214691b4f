"""CPU oracle for the CPSJoin self-join path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package imports this.  Allowed callers: tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference).
"""
