"""The reference's OWN tests against this repo ("the same test
code compiles against either implementation").

tests/cpp/ref_compat/Makefile compiles /root/reference/proj/tests/
test_schedule.cpp, test_bubblefill.cpp, test_perfmodel.cpp (doctest shim) and acceptance.cpp
criteria 1-6 in place, once against include/ + libpf_b200.so (ours_*) and
once against the reference headers + the compiled reference (ref_*).  Both
must pass with identical assertion counts."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "ref_compat", "_bin")
SHIM = os.path.join(ROOT, "tests", "cpp", "ref_compat")


def run(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (make -C tests/cpp/ref_compat where /root/reference exists)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("suite", ["test_schedule", "test_bubblefill", "test_perfmodel"])
def test_reference_unit_tests_pass_against_this_library(suite):
    rc, out = run(f"ours_{suite}")
    assert rc == 0, out[-3000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| 0 failed; assertions: (\d+) \| 0 failed", out)
    assert m and int(m.group(1)) >= 13 and int(m.group(3)) >= 100, out[-1000:]
    rc_ref, out_ref = run(f"ref_{suite}")
    assert rc_ref == 0, out_ref[-3000:]
    # identical test cases and assertion counts on both implementations
    assert out.strip().splitlines()[-1] == out_ref.strip().splitlines()[-1]


def test_reference_acceptance_criteria_1_to_6_pass_against_this_library():
    for impl in ("ours", "ref"):
        rc, out = run(f"{impl}_acceptance_1_6")
        assert rc == 0, out
        assert len(re.findall(r"^\[PASS\] criterion [1-6]:", out, flags=re.M)) == 6, out


def test_doctest_shim_reports_failures(tmp_path):
    """Negative control: a failing CHECK, a REQUIRE that stops its case and
    a missed CHECK_THROWS_AS all fail the run."""
    src = tmp_path / "neg.cpp"
    src.write_text("""
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>
#include <stdexcept>
TEST_CASE("fails") {
    CHECK(1 + 1 == 3);
    CHECK(2.0 == doctest::Approx(2.1));
    CHECK_THROWS_AS((void)0, std::invalid_argument);
    REQUIRE(false);
    CHECK(true);
}
TEST_CASE("subcases run one at a time") {
    static int seen = 0;
    SUBCASE("a") { ++seen; }
    SUBCASE("b") { ++seen; }
    CHECK(seen >= 1);
}
""")
    exe = tmp_path / "neg"
    subprocess.run(["g++", "-std=c++20", "-I", SHIM, str(src), "-o", str(exe)], check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True)
    assert p.returncode == 1
    assert "test cases: 2 | 1 passed | 1 failed" in p.stdout
    assert "assertions: 6 | 4 failed" in p.stdout, p.stdout
