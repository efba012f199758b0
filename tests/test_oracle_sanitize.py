"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (a
sanitizer build of the CPU checker). tests/sanitize/oracle_sanitize_main.c calls
every entry point of oracle/hm_oracle.c on small trees with empty and ragged
leaves, rank-0 levels and nodes, depth 0 and 1, and checks each structured
product against the oracle's dense matrix; built without OpenMP (the sanitizers
and libgomp's thread pool do not mix), so the loops run serially."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_clean_under_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_sanitize")
    cmd = ["gcc", "-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
           "-fno-sanitize-recover=all", "-ffp-contract=off", "-Wall", "-Wno-unknown-pragmas",
           "-I", os.path.join(ROOT, "oracle"),
           os.path.join(ROOT, "tests", "sanitize", "oracle_sanitize_main.c"),
           os.path.join(ROOT, "oracle", "hm_oracle.c"), "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "runtime error" not in r.stderr, r.stderr[-4000:]
    assert "oracle sanitize: clean" in r.stdout
