"""Host build of the device log/sin/cos replicas (csrc/emc_libm.h) against
the system glibc, on the transport argument distributions (see
tests/native/libm_check.c).  The same source compiles for sm_100a with
__dmul_rn/__dadd_rn/__fma_rn, which are the identical IEEE operations; the
device side is checked by tests/test_gpu_parity.py."""

import os
import subprocess

from conftest import ROOT


def test_replica_bit_exact_vs_glibc(tmp_path):
    exe = str(tmp_path / "libm_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "libm_check.c"), "-lm"], check=True)
    out = subprocess.run([exe, "4000000", "11"], capture_output=True, text=True,
                         env=dict(os.environ, OMP_NUM_THREADS="4"))
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout
