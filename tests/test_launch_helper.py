"""The multi-GPU tests' torchrun launcher (tests/launch.py): a rendezvous-port collision
(EADDRINUSE) is retried with a freshly drawn port; other failures are returned as they are."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch import run_torchrun  # noqa: E402

# fails with EADDRINUSE on its first run, succeeds on the second; echoes the port it was given
SCRIPT = """
import os, sys
flag = sys.argv[1]
port = [a for a in sys.argv if a.startswith("--master-port=")][0]
if not os.path.exists(flag):
    open(flag, "w").close()
    sys.stderr.write("DistNetworkError: EADDRINUSE, address already in use\\n")
    sys.exit(1)
print(port)
"""


def test_retries_on_port_collision():
    with tempfile.TemporaryDirectory() as d:
        flag = os.path.join(d, "seen")
        cmd = [sys.executable, "-c", SCRIPT, flag, "--master-port=1"]
        r = run_torchrun(cmd, capture_output=True, text=True, timeout=60)
        assert r.returncode == 0
        port = int(r.stdout.strip().split("=")[1])
        assert 1024 <= port <= 65535  # redrawn, not the placeholder


def test_other_failures_are_not_retried():
    with tempfile.TemporaryDirectory() as d:
        count = os.path.join(d, "count")
        script = ("import sys; open(sys.argv[1], 'a').write('x'); "
                  "sys.stderr.write('some other error'); sys.exit(3)")
        r = run_torchrun([sys.executable, "-c", script, count, "--master-port=1"],
                         capture_output=True, text=True, timeout=60)
        assert r.returncode == 3
        assert open(count).read() == "x"
