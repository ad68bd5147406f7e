"""The drop-in proof: the unmodified reference scheduler (oracle/_ref/libref.so) with
libgplan_shim.so interposed reproduces the reference's golden plans exactly, with
every seam call served by the B200 engine."""
import json
import os
import subprocess
import sys

import pytest

from common import ROOT, golden

pytestmark = pytest.mark.gpu
SHIM = os.path.join(ROOT, "paper_2511_00796_b200", "libgplan_shim.so")
REF = os.path.join(ROOT, "oracle", "_ref", "libref.so")


@pytest.mark.skipif(not (os.path.exists(SHIM) and os.path.exists(REF)),
                    reason="libgplan_shim.so / libref.so not built (need /root/reference at build time)")
def test_reference_scheduler_on_engine_matches_golden():
    keys = sorted(golden("schedules.json"))
    env = dict(os.environ, LD_PRELOAD=SHIM)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dropin_driver.py"), *keys],
                       capture_output=True, text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == len(keys)
    for line in lines:
        g = golden("schedules.json")[line["key"]]
        assert line["plan"] == g["plan"], line["key"]
        assert line["trace"] == g["trace"], line["key"]
        assert line["engine_calls"] > 0
