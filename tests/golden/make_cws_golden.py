"""CWS1 fixtures written by the REFERENCE's own `save_sphere`.

    python tests/golden/make_cws_golden.py

Imports feclab from /root/reference (read-only, this container only) and
writes tests/golden/ref_ca64_r1.cws (CA-polar(64,16)+CRC-11, radius 1) and
tests/golden/ref_ca256_r3.cws (CA-polar(256,16)+CRC-11, radius 3, the
criterion-1 sphere of 538 members; reference tests/test_acceptance.py:51-71).
tests/test_patterns.py checks that this package reads them identically and
writes byte-identical files.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from feclab.codebook import build_ca_polar_code  # noqa: E402
from feclab.wsphere import build_sphere, save_sphere  # noqa: E402

for name, n, k, r in (("ref_ca64_r1", 64, 16, 1), ("ref_ca256_r3", 256, 16, 3)):
    s = build_sphere(build_ca_polar_code(n, k), r)
    save_sphere(s, os.path.join(HERE, name + ".cws"))
    print(name, s.size)
