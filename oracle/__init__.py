"""CPU oracle for the Specx/seqflow GPU execution path.

TEST INFRASTRUCTURE ONLY.  This package is the parity checker and the CPU
baseline; it is never on the product path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product package
``paper_2308_15964_b200`` never imports it and fails loudly when its CUDA
library is missing.

Contents (each module cites the reference file:line it restates):

* ``stf``      -- the reference's sequential-task-flow runtime restated for
                  host worker threads (slot grouping, pending counters,
                  commutative guards, release, FIFO/priority schedulers,
                  trace events, successor edges).
* ``bodies``   -- numpy/scipy FP64 tile bodies (GEMM, SYRK, TRSM, POTRF) and
                  the particle P2P body.  The reference has no tile bodies
                  (SURVEY.md §2 last row), so these are a restatement of the
                  standard BLAS/LAPACK definitions; numeric parity for them is
                  pinned only by golden vectors generated through the real
                  reference engine (tests/golden/make_golden.py).
* ``programs`` -- the insertion loops for tiled DGEMM, right-looking tiled
                  Cholesky and the particle graph, plus the static successor
                  relation (reference tests/conftest.py:160-181).
* ``lru``      -- the reference's independent LRU model
                  (reference tests/test_device.py:37-54) and the arena
                  first-fit/LRU allocator (reference src/device.py:78-264).
* ``inputs``   -- seeded splitmix64 input generators shared bit-for-bit with
                  the CUDA generator kernels.
"""
