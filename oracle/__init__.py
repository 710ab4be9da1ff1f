"""TEST INFRASTRUCTURE ONLY.

CPU oracle for the B200 executor: a numpy restatement of the reference
`qvirt` hot path (kernels, backend reductions, DDCL / MC-VQE drivers) plus
the reference's dense-matrix oracle.  Only `tests/`, `__graft_entry__.smoke()`
and bench.py's `cpu_baseline` / `--impl reference` legs may import it, and
only as the checker or the timed CPU baseline -- never as the product path.
"""
