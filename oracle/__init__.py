"""CPU oracle for LUT-GEMM -- TEST INFRASTRUCTURE ONLY (see bcq_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the CUDA path.
"""
from .bcq_oracle import *  # noqa: F401,F403
from .bcq_oracle import __all__  # noqa: F401
