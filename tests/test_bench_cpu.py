"""bench.py's reference arm (--impl reference) on CPU: it times the reference
itself (oracle/_ref/libgs_ref.so) when that library is present, else the
restated port, with the GPU arm's config dict, reports the host CPU model /
physical core count, and never maps the product library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = """
import sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "{w}", "--steps", "2", "--warmup", "3"]
sys.path.insert(0, {root!r})
import bench
bench.main()
print("MAPPED", open("/proc/self/maps").read().count("libgs_b200"))
"""


def run(w):
    out = subprocess.run([sys.executable, "-c", PROBE.format(w=w, root=ROOT)], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    return json.loads(lines[-2]), int(lines[-1].split()[1])


def test_reference_arm_is_product_free_and_shares_config():
    import bench
    line, mapped = run("c1")
    assert mapped == 0
    assert line["impl"] == "reference" and line["config"] == bench.config_for("c1", 1, 1)
    from oracle import ref
    assert line["cpu_baseline"]["kind"] == ("reference" if ref.available() else "port")
    assert line["cpu_baseline"]["cpu_model"]
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
