"""The checked build (-m gpu): libntbc_checked.so = libntbc.so compiled with NTBC_CHECKS=1 -- every computed
shared-memory / TMEM / global index of the fused and pack kernels bounds-checked (a failure traps), shared
memory poisoned with NaN patterns before use -- run over ragged shapes, odd grid resolutions, extreme head
layouts, naive and conservative models, row shards and the pack kernel, each word compared with the oracle,
under five schedules (work groups per CTA 2/3/4/8, static and dynamic unit scheduling): a race or an
uninitialised read shows up as a trap, an oracle mismatch, or words that depend on the schedule.  It stands
in for compute-sanitizer (memcheck / racecheck / initcheck), which this GPU pool refuses
(profiles/r02c_compute_sanitizer_refused.log)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(env_extra, tag):
    lib = os.path.join(ROOT, "paper_2407_09543_b200", "libntbc_checked.so")
    if not os.path.exists(lib):
        pytest.fail("libntbc_checked.so is not built (make -C paper_2407_09543_b200/csrc)")
    env = dict(os.environ, NTBC_LIB="libntbc_checked.so", **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_run.py"), tag], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    line = [l for l in out.stdout.splitlines() if l.startswith("OK")]
    assert line, out.stdout[-2000:]
    return line[-1].split()[-1]


def test_checked_build_all_schedules_agree():
    digests = {}
    for tag, env in (("nwg8", {"NTBC_NWG": "8"}), ("nwg4", {"NTBC_NWG": "4"}), ("nwg3", {"NTBC_NWG": "3"}),
                     ("nwg2", {"NTBC_NWG": "2"}), ("static", {"NTBC_STATIC_SCHED": "1"})):
        digests[tag] = _run(env, tag)
    assert len(set(digests.values())) == 1, digests
