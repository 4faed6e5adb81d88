"""The opt-in TS form of the resident-A pair kernel (VNM_TC3_TS=1: A copied once into TMEM by tcgen05.cp and read
from there by the sparse MMAs) against the oracle.  The switch is read once per process, so the checks run in a
child process with it set; the same sampled / full comparisons as tests/test_gpu_spmm.py."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import torch
from tests.test_gpu_spmm import sampled_check, make, gpu_y, assert_within
import oracle
# DeiT-S qkv / fc1 at full size (T = 50,432 = 197 x 256), bf16 Y, sampled outputs; a small full-output case
sampled_check(1152, 384, 5, 50432, seed=7, out_dtype=torch.bfloat16, tc=True)
sampled_check(1536, 384, 5, 50432, seed=8, tc=True)
W, XT, Wm = make(768, 384, 64, 5, 8192 + 256, seed=9)
Yref, Aref = oracle.gemm_ref(XT, Wm)
assert_within(gpu_y(W, XT, 64, 5, 8192 + 256, tc=True), Yref, Aref)
print("ts ok")
"""


def test_tc3_ts_form_matches_oracle():
    env = dict(os.environ, VNM_TC3_TS="1", PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ts ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
