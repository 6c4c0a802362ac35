"""The seeded generator's scene kinds against the paper's per-motion-level pruning (§6: codec-guided
pruning removes 50 %, 27 % and 13 % of the visual tokens of low-, medium- and high-motion videos), measured with
the oracle on fresh seeds.  These are generator properties (UCF-Crime statistics reproduced on synthetic
metadata), not a parity pin: each kind must land within 10 points of its target kept fraction."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import calibrate_synth  # noqa: E402


@pytest.mark.parametrize("scene", ["static", "low", "medium", "high", "traffic"])
def test_scene_kept_fraction_band(ref, scene):
    streams, frames = (4, 40) if scene == "traffic" else (8, 48)
    got = calibrate_synth.kept_fraction(scene, streams=streams, frames=frames, seed0=11)
    target = calibrate_synth.TARGETS[scene]
    assert abs(got - target) <= 0.10, (scene, got, target)


def test_motion_levels_ordered(ref):
    k = {sc: calibrate_synth.kept_fraction(sc, streams=6, frames=48, seed0=5) for sc in ("low", "medium", "high")}
    assert k["low"] < k["medium"] < k["high"], k
