"""CPU oracle for the GSpaRC render/train hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2511_22793_b200`) may import this package.  It is imported by
`tests/`, by `__graft_entry__.smoke()` (as the checker) and by `bench.py`'s
CPU-baseline leg / `--impl reference` arm (as the timed CPU reference).

The oracle is a NumPy restatement of the reference package `rfsplat`
(`/root/reference/pkg/src/rfsplat`), pinned against golden vectors produced by
the real reference (`tests/golden/make_golden.py` -> `tests/golden/*.npz`).
"""

from .rfsplat_oracle import *  # noqa: F401,F403
