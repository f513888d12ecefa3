"""CPU oracle for the VarStream search path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import anything under ``oracle/``; the product
package (``paper_2010_02164_b200``) never does and fails loudly when its CUDA
library is missing.

Parity pinning: ``tests/golden/*.json`` were produced by running the
UNMODIFIED reference (``/root/reference/pkg/src/beambatch``) in the build
container (``oracle/gen_golden.py``); ``tests/test_oracle_golden.py`` checks
this restatement against every one of them.
"""
