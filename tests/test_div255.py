"""The fused NV12 kernel replaces the IEEE division v / 255 by q = v * RN(1/255) plus one fma residual correction.
This pins that identity (bit-exact for every fp32 v in [0, 512]) on a strided sample of all floats; the full
exhaustive run is `scripts/check_div255.c` with stride 1."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_div255_identity(tmp_path):
    exe = tmp_path / "check_div255"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), os.path.join(ROOT, "scripts", "check_div255.c"),
                    "-lm"], check=True)
    out = subprocess.run([str(exe), "97"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout


def test_norm_bf16_guarded_reciprocal(tmp_path):
    """The NV12 normalisation's bf16((t - mean) / std) through q = RN(a * RN(1/std)) with the exact division only
    when q is within 8 steps of a bf16 rounding midpoint: equal to the oracle's fp32 division + RNE on a strided
    sample of every fp32 a in [-4, 4] for 16 std values (the full sweep is scripts/check_norm_bf16.c stride 1).
    Without the guard the same sample has mismatches, so the check is sensitive to it."""
    src = os.path.join(ROOT, "scripts", "check_norm_bf16.c")
    for extra, want_bad in (([], False), (["-DNOGUARD"], True)):
        exe = tmp_path / ("cnb" + "".join(extra))
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", *extra, "-o", str(exe), src, "-lm"], check=True)
        out = subprocess.run([str(exe), "211", "8"], capture_output=True, text=True)
        assert (out.returncode != 0) == want_bad, out.stdout
        assert ("mismatches 0" in out.stdout) != want_bad
