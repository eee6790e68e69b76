"""Which NVML NVLink byte counters does this GPU expose (per link)?"""
import pynvml as n

n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(0)
fields = {k: getattr(n, k) for k in dir(n) if k.startswith("NVML_FI_DEV_NVLINK") and
          any(x in k for x in ("THROUGHPUT", "COUNT_XMIT_BYTES", "COUNT_RCV_BYTES"))}
for name, fid in sorted(fields.items(), key=lambda t: t[1]):
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = n.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, fid, "scope", scope, "ret", v.nvmlReturn, "val", v.value.ullVal)
        except Exception as e:
            print(name, fid, "scope", scope, "exc", type(e).__name__, e)
try:
    print("nvlink state link0", n.nvmlDeviceGetNvLinkState(h, 0))
    print("util counter", n.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0))
except Exception as e:
    print("legacy", type(e).__name__, e)
