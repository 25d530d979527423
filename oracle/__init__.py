"""fp64 CPU oracle for the 3DPIFCM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2002_01981_b200`` never imports it and shares no code
with it.  The arithmetic lives in ``pifcm_oracle.c`` (plain loops, fp64); this
module only marshals numpy arrays through ctypes.

Citations: PAPER:N = /root/reference/PAPER.md line N.
"""
from .oracle import *  # noqa: F401,F403
from .oracle import build_oracle, lib_path  # noqa: F401
