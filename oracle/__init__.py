"""CPU oracle for parity -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_quant_ph_0608239_b200) never imports it and shares no code with it.
"""
from .oracle import Oracle, build_oracle, oracle_lib_path  # noqa: F401
