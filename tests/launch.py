"""torchrun launcher for the multi-GPU tests: picks a free rendezvous port and retries with a new
one when the rendezvous server loses the race for it (EADDRINUSE between probing and binding)."""
import socket
import subprocess


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_torchrun(cmd, attempts=4, **kw):
    """subprocess.run(cmd, **kw) with `--master-port=...` re-drawn on a port collision."""
    r = None
    for _ in range(attempts):
        cmd = [f"--master-port={free_port()}" if a.startswith("--master-port=") else a for a in cmd]
        r = subprocess.run(cmd, **kw)
        out = (r.stdout or "") + (r.stderr or "")
        if r.returncode == 0 or "EADDRINUSE" not in out:
            return r
    return r
