"""CPU oracle for the rational-approximation time stepper.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.
Shares no code with paper_1402_5168_b200/ (the CUDA path).
"""
