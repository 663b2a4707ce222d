"""fp64 CPU oracle for the FD-curvature neural-SDF step.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this package.
The product path (paper_2511_08980_b200) never imports it and shares no code,
constants or helpers with it.
"""
from .fdsdf_oracle import *  # noqa: F401,F403
from .train_oracle import *  # noqa: F401,F403
