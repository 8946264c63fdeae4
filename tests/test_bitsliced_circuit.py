"""CPU: the generated bitsliced S-box circuit is what the generator emits
(which verifies it on all 256 inputs before writing)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generated_sbox_is_current_and_verified():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_bitsliced_sbox.py"), "--check"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
