"""CPU oracle for the MoE-layer hot path — TEST INFRASTRUCTURE ONLY.

routing_ref.py restates the reference's moelab.routing (pkg/src/moelab/routing.py) and
perf.a2a_send_volume; backward_ref.py restates the exact gradient of that forward.
Pinned by tests/test_oracle.py against golden vectors produced by the reference itself.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference legs import
this package; the product package paper_2603_07685_b200 never does.
"""
