"""INTEGRATION.md's code runs as written: the plain ctypes stub (the binding a
reference maintainer would add) and the device-resident snippet are pulled
out of the document and executed against the built library, their outputs
checked against the oracle."""
import os
import random
import re

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _block_after(marker: str) -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    tail = text[text.index(marker):]
    return re.search(r"```python\n(.*?)```", tail, re.S).group(1)


def test_ctypes_stub_runs_as_documented(lib, gpu, orc):
    from paper_1403_7295_b200 import _native

    code = _block_after("**Plain ctypes stub.**").replace("/path/to/libpaes_cuda.so", _native.lib_path())
    rnd = random.Random(33)
    env = {"key": rnd.randbytes(16), "data": rnd.randbytes(100_003)}
    exec(compile(code, "INTEGRATION.md:ctypes-stub", "exec"), env)
    assert env["rc"] == 0
    assert env["out"].raw[: env["n"].value] == orc.encrypt_chunk(env["data"], True, env["key"])


def test_device_snippet_runs_as_documented(paes, gpu, orc):
    import torch

    code = _block_after("## 4. Device-resident use")
    rnd = random.Random(34)
    key, data = rnd.randbytes(16), rnd.randbytes(65_541)
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    dst = torch.empty(len(data) + 16, dtype=torch.uint8, device="cuda")
    env = {"key": key, "src": src, "dst": dst, "nbytes": len(data)}
    exec(compile(code, "INTEGRATION.md:device", "exec"), env)
    torch.cuda.synchronize()
    assert dst[: env["n_out"]].cpu().numpy().tobytes() == orc.encrypt_chunk(data, True, key)
