"""CPU oracle (TEST INFRASTRUCTURE ONLY) — see ``oracle/ring_oracle.py`` and
``oracle/negotiation.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.
"""
from .ring_oracle import *  # noqa: F401,F403
from .ring_oracle import (DEFAULT_FUSION_BYTES, MEMBER_ALIGN_BYTES, CHUNK_QUANTUM_BYTES,  # noqa: F401
                          Entry, FusionBuffer, Traffic)
from . import negotiation  # noqa: F401,E402
