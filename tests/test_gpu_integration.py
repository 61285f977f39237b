"""The reference-side binding (integration/espec/b200.hpp) compiled against
the UNMODIFIED reference headers and core (oracle/_ref/libespec_ref.a, built
from /root/reference/proj by oracle/Makefile) and linked to
libespec_b200.so: generate_b200 and the stage calls (B200Generation) must
reproduce espec::generate's tokens and alpha on the same Model objects, and
raise the reference's CheckError on the fixture where it throws."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "integration_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="integration_check is built where /root/reference exists "
                                                    "(make -C oracle integration) and ships with the repo")
def test_reference_binding_reproduces_generate():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and out["ok"], out
    names = {c["name"]: c for c in out["cases"]}
    assert names["greedy_tree_throws_indep"]["b200_error"] == "sibling candidates exhaust the draft distribution"
    assert names["c1_easyspec"]["tokens"] == 64
