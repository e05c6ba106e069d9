"""CPU oracle for parity tests — TEST INFRASTRUCTURE, never the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package. See ``cacheclip_oracle.py`` for the parity
status (pinned against the reference's own outputs in ``tests/golden/``).
"""
