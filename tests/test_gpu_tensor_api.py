"""torch-facing wrappers: encrypt_tensor / decrypt_tensor on the current stream."""
import os

import pytest

pytestmark = pytest.mark.gpu


def test_tensor_round_trip(paes, gpu, orc):
    import torch

    key = bytes(range(16))  # fixed: the wrong-key check below must not flake on a 1/256 valid trailer
    for n in [0, 5, 16, 4097, 1 << 20]:
        data = os.urandom(n)
        x = torch.frombuffer(bytearray(data + b"\0"), dtype=torch.uint8)[:n].cuda()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ct = paes.encrypt_tensor(x, key)
            pt = paes.decrypt_tensor(ct, key)
        s.synchronize()
        assert ct.cpu().numpy().tobytes() == orc.encrypt_chunk(data, True, key)
        assert pt.cpu().numpy().tobytes() == data
    with pytest.raises(ValueError):
        paes.encrypt_tensor(torch.zeros(16, dtype=torch.uint8), key)  # CPU tensor
    with pytest.raises(paes.PaddingError):
        paes.decrypt_tensor(paes.encrypt_tensor(torch.zeros(40, dtype=torch.uint8, device="cuda"), key),
                            bytes(16))
