"""GPU: the reference's OWN operator and neighbourhood test suites with the B200 module in
the reference's kernel slot (the `kernel_backend` fixture,
/root/reference/pkg/tests/conftest.py:7-11, over backend.py:53-62).

oracle/build_ref.sh packs the unmodified reference package and its tests into
oracle/_ref/refsuite.tar.gz (built here, git-ignored, shipped to the GPU box with the
library); this test unpacks it into a temporary directory and runs
    pytest test_flexops.py test_neighborhood.py -p b200_slot_plugin
in a subprocess, so every flexops / knn_query call of those tests goes through
paper_1803_07289_b200.backend -> the C ABI -> the CUDA kernels (fp64 engine).
"""

import os
import re
import subprocess
import sys
import tarfile

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TARBALL = os.path.join(ROOT, "oracle", "_ref", "refsuite.tar.gz")


@pytest.mark.parametrize("suite", ["test_flexops.py", "test_neighborhood.py"])
def test_reference_suite_through_the_b200_slot(fc, tmp_path, suite):
    if not os.path.exists(TARBALL):
        pytest.skip("oracle/_ref/refsuite.tar.gz not built (oracle/build_ref.sh needs /root/reference)")
    with tarfile.open(TARBALL) as tf:
        tf.extractall(tmp_path, filter="data")
    pkg = tmp_path / "refpkg"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(pkg), os.path.join(ROOT, "tests", "ref_suite"), ROOT,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "b200_slot_plugin", "-m", "not slow",
           "-p", "no:cacheprovider", str(pkg / "tests" / suite)]
    res = subprocess.run(cmd, cwd=str(pkg), env=env, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert "flexconv kernel slot: paper_1803_07289_b200.backend" in out, out[-3000:]
    assert res.returncode == 0, out[-6000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) > 0, out[-3000:]
    print(f"{suite}: {m.group(0)} with the B200 module in the kernel slot")
