"""The C oracle under AddressSanitizer + UndefinedBehaviorSanitizer: tests/sanitize/oracle_asan_driver.c
drives every oracle entry point (score, compact incl. capacity truncation, temporal patches, out-of-place and paged
KV refresh in fp32 and bf16/M-RoPE, NV12 preprocessing, MV rasterisation, similar histogram, RoPE, patch fields) on
a C1-shaped stream and a ragged geometry; any sanitizer report aborts it (-fno-sanitize-recover=all)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_asan_ubsan(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "oracle_asan")
    cmd = [gcc, "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-ffp-contract=off",
           "-I", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "codecsight_ref.c"),
           os.path.join(ROOT, "tests", "sanitize", "oracle_asan_driver.c"), "-lm", "-o", exe]
    b = subprocess.run(cmd, capture_output=True, text=True)
    if b.returncode != 0 and "asan" in (b.stderr or "").lower():
        pytest.skip("sanitizer runtime not available: " + b.stderr[-300:])
    assert b.returncode == 0, b.stderr[-3000:]
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "oracle sanitizer driver: ok" in r.stdout
    assert "runtime error" not in r.stderr and "AddressSanitizer" not in r.stderr
