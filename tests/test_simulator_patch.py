"""CPU check of shim/patches/simulator_b200.patch (the C5 loop's host
simulator): tools/sim_compare.sh plans C5 steps with the reference planner
and prints every run_step result (events, segments, releases) for the three
cut modes, once with the reference's simulator.cpp and once with the patched
copy; the two outputs must be byte-identical. Needs the reference sources
(build time only) and `make shim` / `make -C oracle ref`."""
import pathlib
import subprocess

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]


def test_patched_simulator_matches_reference():
    if not pathlib.Path("/root/reference/proj/src/simulator.cpp").exists():
        pytest.skip("reference sources not present")
    if not (REPO / "build/shim/simulator_b200.cpp").exists() or not (REPO / "oracle/_ref/obj/simulator.o").exists():
        pytest.skip("make shim / make -C oracle ref not run")
    p = subprocess.run(["bash", "tools/sim_compare.sh", "2"], cwd=REPO, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "identical" in p.stdout
