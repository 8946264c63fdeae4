"""Performance floors on the B200, so a regression in the hot kernels fails the
suite instead of only moving the bench number.  Device-resident, CUDA-event
timed, best of 5 launches.  Floors sit ~15-20 % below the measured rates
(869 / 864 / 852 GB/s at 1965 MHz) and scale with the SM clock read through
NVML right after the launches: the kernels are bound by the shared-memory
lookup pipe, whose rate is proportional to the clock, so a box held at a
lower clock (power cap) is not mistaken for a regression."""
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


def _clock_scale(torch, busy) -> float:
    """SM clock under load / 1965 MHz (the clock the floors were set at), at
    most 1: `busy` queues ~0.1 s of kernels, NVML is read while they run."""
    try:
        import pynvml

        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(0)  # CUDA ordinal 0 != NVML index under CUDA_VISIBLE_DEVICES
            h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")
            busy()
            mhz = max(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM) for _ in range(5))
            torch.cuda.synchronize()
        finally:
            pynvml.nvmlShutdown()
        return min(1.0, max(0.3, mhz / 1965.0))
    except Exception:  # no NVML: fixed floors
        torch.cuda.synchronize()
        return 1.0


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
    def busy():
        for _ in range(20):
            paes.ecb_device(0, a.data_ptr(), b.data_ptr(), n, rk, 0, s)

    k = _clock_scale(torch, busy)
    print(f"clock scale {k:.3f}")
    assert enc >= 720 * k, f"encrypt {enc:.1f} GB/s (clock scale {k:.2f})"
    assert dec >= 720 * k, f"decrypt {dec:.1f} GB/s (clock scale {k:.2f})"
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
    assert bat >= 680 * k, f"batch {bat:.1f} GB/s (clock scale {k:.2f})"
    del a, b
    torch.cuda.empty_cache()
