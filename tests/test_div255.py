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
