#!/usr/bin/env python
"""Device-local timing of the ring's wire format on one GPU: the strided core
copy (g4_copy_payload_cores) against a contiguous copy of the whole staged
payloads, and the receiver-side halo rebuild (g4_fill_halo).  Measurement
tool (peer copies over NVLink need two GPUs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2105_00027_b200 import _lib, tensor as T  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def sweep():
    """BASELINE config 5: one ring message of 64 KB - 64 MB (one walker's payload
    cores, N = 45 ... 1448), both wire formats, complex128 and complex64:
    time per message including launch latency (device-local copy engine)."""
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    print("message sweep (device-local; one payload per message):")
    for n in (45, 64, 128, 256, 362, 512, 724, 1024, 1448):
        for dt, code, eb in ((torch.complex128, _lib.G4_C128, 16), (torch.complex64, _lib.G4_C64, 8)):
            shape = (1,) + T.staged_shape(n, dt)
            src = torch.randn(shape, dtype=dt, device="cuda")
            dst = torch.empty_like(src)
            full = src.numel() * src.element_size()
            core = 2 * n * n * eb
            t_core = timed(lambda: _lib.check(lib.g4_copy_payload_cores(dst.data_ptr(), src.data_ptr(), 1, n, code, st)))
            t_full = timed(lambda: _lib.check(lib.g4_copy_async(dst.data_ptr(), src.data_ptr(), full, st)))
            ptrs = _lib.ptr_array([dst[0].data_ptr()])
            t_halo = timed(lambda: _lib.check(lib.g4_fill_halo(ptrs, 1, n, code, st)))
            print(f"  N={n:5d} {'c128' if eb == 16 else 'c64 '} cores {core / 1e6:8.3f} MB {t_core * 1e6:8.1f} us "
                  f"({core / t_core / 1e9:5.0f} GB/s) + halo {t_halo * 1e6:6.1f} us | staged {full / 1e6:8.3f} MB "
                  f"{t_full * 1e6:8.1f} us ({full / t_full / 1e9:5.0f} GB/s)", flush=True)


def main():
    if "--sweep" in sys.argv:
        return sweep()
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    for n, B in ((512, 8), (1024, 8), (4608, 2)):
        shape = (B,) + T.staged_shape(n)
        src = torch.randn(shape, dtype=torch.complex128, device="cuda")
        dst = torch.empty_like(src)
        full = src.numel() * 16
        core = B * 2 * n * n * 16
        t_core = timed(lambda: _lib.check(lib.g4_copy_payload_cores(dst.data_ptr(), src.data_ptr(), B, n,
                                                                     _lib.G4_C128, st)))
        t_full = timed(lambda: _lib.check(lib.g4_copy_async(dst.data_ptr(), src.data_ptr(), full, st)))
        ptrs = _lib.ptr_array([dst[i].data_ptr() for i in range(B)])
        t_halo = timed(lambda: _lib.check(lib.g4_fill_halo(ptrs, B, n, _lib.G4_C128, st)))
        print(f"N={n} B={B}: core copy {core / 1e6:.1f} MB in {t_core * 1e6:.1f} us ({core / t_core / 1e9:.0f} GB/s); "
              f"full staged copy {full / 1e6:.1f} MB in {t_full * 1e6:.1f} us ({full / t_full / 1e9:.0f} GB/s); "
              f"halo rebuild {t_halo * 1e6:.1f} us", flush=True)


if __name__ == "__main__":
    main()
