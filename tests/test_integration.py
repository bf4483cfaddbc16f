"""The maintainer-side C++ shim (integration/pipeline_b200.hpp, embedded in INTEGRATION.md)
compiled against the reference's own headers and linked with both the reference's sources
(oracle/_ref) and the B200 library: integration/_build/demo runs the reference's Pipeline /
spaqr_factorize / cgls / factor files next to the B200 bindings in one process."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "integration", "_build", "demo")


def test_integration_md_embeds_the_compiled_shim():
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    hpp = open(os.path.join(ROOT, "integration", "pipeline_b200.hpp")).read()
    block = md.split("```cpp\n", 1)[1].split("```", 1)[0]
    assert block.strip() == hpp.strip()


@pytest.mark.skipif(not os.path.exists(DEMO), reason="integration demo not built (needs /root/reference)")
def test_shim_refuses_without_gpu():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([DEMO, "/tmp"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CHECK no_gpu_refuses ok" in r.stdout


@pytest.mark.gpu
def test_shim_matches_reference_on_gpu(tmp_path):
    assert os.path.exists(DEMO), "integration/_build/demo missing: build() in the container builds it"
    r = subprocess.run([DEMO, str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr
