"""The C++ drop-in: reference-style assertions (tests/cpp/test_kfac_dropin.cpp)
compiled against include/pipefill/kfac/*.hpp and linked against the product
library — the source a reference caller writes, running on the B200."""
import os
import subprocess

import pytest

from conftest import HAS_GPU, ROOT

LIB = os.path.join(ROOT, "paper_2211_14133_b200", "_lib")
BIN = os.path.join(LIB, "test_kfac_dropin")


def test_dropin_binary_built_and_symbols_exported():
    assert os.path.exists(BIN), "run __graft_entry__.build() (make -C paper_2211_14133_b200)"
    out = subprocess.run(["nm", "-DC", os.path.join(LIB, "libpf_b200.so")], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("pipefill::kfac::curvature_factors(", "pipefill::kfac::cholesky_spd_inverse(",
                "pipefill::kfac::precondition(", "pipefill::kfac::ngd_step(",
                "pipefill::kfac::KfacState::update_factors(", "pipefill::kfac::KfacState::refresh_inverses(",
                "pipefill::build_schedule(", "pipefill::assign_works(", "pipefill::enumerate_kfac_works("):
        assert sym in out, sym


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device behaviour")
def test_dropin_fails_loudly_without_device():
    r = subprocess.run([BIN], capture_output=True, text=True)
    assert r.returncode != 0
    assert "no usable sm_100" in r.stderr + r.stdout


@pytest.mark.gpu
def test_dropin_reference_assertions_pass_on_b200():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
