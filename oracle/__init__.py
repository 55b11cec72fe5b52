"""CPU oracle (test infrastructure only) — see oracle/oracle.py and oracle/vm_oracle.h."""
from .oracle import *  # noqa: F401,F403
from .oracle import Oracle, OracleError, available, Contraction, Field, MarchConfig, Packed  # noqa: F401
