"""Performance floors on the B200, so a regression in the hot kernels fails the
suite instead of only moving the bench number.  Device-resident, CUDA-event
timed, best of 5 launches.  Floors sit ~15-20 % below the measured rates
(869 / 864 / 835 GB/s at 1965 MHz), leaving room for clock variation."""
import pytest

pytestmark = pytest.mark.gpu
GiB = 1 << 30


def _best_gbs(torch, fn, nbytes, reps=5):
    s = torch.cuda.current_stream()
    fn()
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def test_kernel_throughput_floors(paes, gpu):
    import torch

    n = 4 * GiB
    rk = paes.round_keys(bytes(range(16)))
    a = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    b = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    paes.counter_fill_device(7, 0, n, a.data_ptr())
    s = torch.cuda.current_stream().cuda_stream
    enc = _best_gbs(torch, lambda: paes.ecb_device(0, a.data_ptr(), b.data_ptr(), n, rk, 0, s), n)
    dec = _best_gbs(torch, lambda: paes.ecb_device(1, b.data_ptr(), a.data_ptr(), n, rk, 0, s), n)
    assert enc >= 720, f"encrypt {enc:.1f} GB/s"
    assert dec >= 720, f"decrypt {dec:.1f} GB/s"
    # batch: 256 messages of 4 MiB - 16 B, per-message keys, one launch
    L = (4 << 20) - 16
    lens = [L] * 256
    offs = [i * (4 << 20) for i in range(256)]
    rks = b"".join(paes.round_keys(bytes([i % 256] * 16)) for i in range(256))
    plan = paes.BatchPlan(0, offs, offs, lens, rks, True)
    try:
        bat = _best_gbs(torch, lambda: plan.run(a.data_ptr(), b.data_ptr(), s), L * 256)
    finally:
        plan.close()
    assert bat >= 680, f"batch {bat:.1f} GB/s"
    del a, b
    torch.cuda.empty_cache()
