"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the B200 backend.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and only
as the checker or the reported CPU baseline -- never on the product path
(the product package has no import of it, and fails loudly without its CUDA
library).

* ``oracle.dsl``    -- restatement of the reference's serial semantics for
  task-body programs (eval_kernel, ReadView clamping, mapper images) in
  numpy; pinned against the reference itself by tests/test_oracle.py and by
  the golden fixtures in tests/golden/ (generated from the reference by
  tests/golden/make_golden.py).
* ``oracle.native`` -- ctypes loader for ``cq_oracle.c`` (SAXPY, wave step,
  N-body, matmul rows) built into ``oracle/_build/liboracle.so``.
"""
