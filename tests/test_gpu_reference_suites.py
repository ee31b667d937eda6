"""The reference's own unit suites (proj/tests/test_{tensor,layers,netgraph,pipeline,malis}.cpp)
run against the drop-in: built by __graft_entry__.build() with tests/cpp/redirect.hpp
force-included, so every call the suites make of conv/pool/relu/upconv/mergecrop/softmax
forward, im2col, gemm, the float backward functions, softmax_loss, sgd_step, process<float>,
mirror_pad, normalize_image<float>, NetRunner<float> and the MALIS functions runs on the B200
(double-precision backward/NetRunner/process calls stay on the reference; the count is printed).
The suites' assertions are the reference's own -- oracles, finite-difference gradient checks,
message checks -- over the doctest subset in tests/cpp/doctest_shim."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SUITES = ("test_tensor", "test_layers", "test_netgraph", "test_pipeline", "test_malis")
# lower bounds on the calls each suite makes of the B200 side (guards against a silent
# redirect regression; the exact counts are in the output)
MIN_GPU_CALLS = {"test_tensor": 10, "test_layers": 15, "test_netgraph": 5, "test_pipeline": 200, "test_malis": 30}


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_dropin(suite):
    exe = os.path.join(ROOT, "build", "ref_" + suite)
    if not os.path.exists(exe):
        pytest.skip(f"build/ref_{suite} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-8000:] + r.stderr[-2000:]
    m = re.search(r"\| (\d+) passed \| (\d+) failed \| assertions", r.stdout)
    assert m and int(m.group(2)) == 0 and int(m.group(1)) > 0
    g = re.search(r"calls on the B200 drop-in: (\d+)", r.stdout)
    assert g and int(g.group(1)) >= MIN_GPU_CALLS[suite], r.stdout[-2000:]
