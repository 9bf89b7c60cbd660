"""pytest plugin: install the B200 kernel module in the reference package's backend slot.

Loaded with `-p b200_slot_plugin` when tests/test_gpu_ref_suite.py runs the REFERENCE's own
test files (unpacked from oracle/_ref/refsuite.tar.gz).  The reference selects its kernels
through `flexconv.backend` (/root/reference/pkg/src/flexconv/backend.py:34-62): `_active` is
what every operator calls, and the `kernel_backend` fixture (tests/conftest.py:7-11)
parametrises over "native" and "reference".  After this plugin:
  * `_active` (the default every test uses) and "native" are paper_1803_07289_b200.backend;
  * "reference" stays the reference's numpy kernels, so the reference's cross-backend tests
    (test_flexops.py:71-81, test_neighborhood.py:84-106) compare the B200 module with them.
"""

import sys

import paper_1803_07289_b200.backend as b200_backend
from flexconv import backend as ref_backend

ref_backend._native = b200_backend
ref_backend._active = b200_backend
sys.stderr.write(f"flexconv kernel slot: {ref_backend.active().__name__} "
                 f"(native -> {ref_backend.get('native').__name__})\n")
