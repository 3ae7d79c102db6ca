"""Gauss-Gram operand feeds (csrc/gram_tc.cu, template CV): S / D formed in
shared memory (PS_GAUSS_CONV=1) must hand the tensor cores the same fp16
operands as the streamed S / D planes (gauss_planes_kernel), i.e. identical
PLV / iPLV / ciPLV bits, for the CTA-pair and the one-CTA kernels; one-trial
cases also against an fp64 restatement (1e-5, the split tolerance).  Environment switches are read
once per process, hence the subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_gauss_smem_feed_bit_identical():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "gauss_conv_check.py")], capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-2000:])
    assert "gauss_conv_check OK" in out.stdout
