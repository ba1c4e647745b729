"""CPU oracle for the B200 PCG-sampler path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package `priorcg` (arXiv 1810.12437,
/root/reference/pkg/src/priorcg) on the beta-draw hot path, each function
citing the reference file:line it follows.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline / reference arms may import this package, and
only as the checker or the timed CPU baseline: the product package
`paper_1810_12437_b200` never imports it.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports priorcg in the build
container; the fixtures are committed), bit-for-bit where the reference's
arithmetic is replayed with the same numpy calls and RNG stream.
"""
