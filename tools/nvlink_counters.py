"""NVLink byte counters through NVML field values (KiB, per GPU, all links):
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (and the RAW variants). Used by
tools/bench_a2a.py to report the bytes the fused dispatch/combine moved over
NVLink; `python tools/nvlink_counters.py` probes them with a 1 GiB P2P copy."""
from __future__ import annotations


def _nvml():
    import pynvml
    pynvml.nvmlInit()
    return pynvml


def read(index: int) -> dict:
    """{'tx': bytes, 'rx': bytes, 'raw_tx': bytes, 'raw_rx': bytes} (None when unsupported)."""
    nv = _nvml()
    h = nv.nvmlDeviceGetHandleByIndex(index)
    ids = [getattr(nv, n, None) for n in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX",
                                         "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
                                         "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX",
                                         "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX")]
    out = {}
    for key, fid in zip(("tx", "rx", "raw_tx", "raw_rx"), ids):
        out[key] = None
        if fid is None:
            continue
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [fid])[0]
            if v.nvmlReturn == 0:
                out[key] = int(v.value.ullVal) * 1024  # KiB -> bytes
        except Exception:
            pass
    return out


def delta(a: dict, b: dict) -> dict:
    return {k: (b[k] - a[k]) if a.get(k) is not None and b.get(k) is not None else None
            for k in a}


if __name__ == "__main__":
    import torch
    n = torch.cuda.device_count()
    x = torch.empty(1 << 29, dtype=torch.int16, device="cuda:0")  # 1 GiB
    print("devices", n)
    before = [read(i) for i in range(n)]
    if n > 1:
        y = torch.empty_like(x, device="cuda:1")
        for _ in range(4):
            y.copy_(x)
        torch.cuda.synchronize()
    after = [read(i) for i in range(n)]
    for i in range(n):
        print(i, before[i], delta(before[i], after[i]))
