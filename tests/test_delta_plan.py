"""CPU check of the Witt-carry kernel's index algebra (qfs_delta_mma.cuh): tools/check_delta_plan.cpp replays, with indices only,
what k_delta_mma does for every phase of every supported prime and demands that entries and guard zeros cover every word of the
quad's Delta array exactly once, at the offset the matrix builder expects (qfs_shape.cuh)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_delta_plan_covers_delta_exactly_once(tmp_path):
    exe = str(tmp_path / "check_delta_plan")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", exe, os.path.join(ROOT, "tools", "check_delta_plan.cpp")])
    out = subprocess.run([exe], capture_output=True, text=True)
    sys.stdout.write(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count(": ok") == 10
