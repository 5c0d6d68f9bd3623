"""Test infrastructure only: CPU checker for the AMSP data plane and the
compiled reference planner. Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference legs may import this package."""
