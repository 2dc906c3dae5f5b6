"""Probe (context only): which NVML NVLink counters this driver exposes on this GPU."""
import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
print("driver", nv.nvmlSystemGetDriverVersion(), "name", nv.nvmlDeviceGetName(h))
for l in range(18):
    try:
        st = nv.nvmlDeviceGetNvLinkState(h, l)
    except Exception as e:  # noqa: BLE001
        st = f"err {e}"
    print("link", l, "state", st)
names = ["NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES",
         "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
         "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX"]
for name in names:
    fid = getattr(nv, name)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, "scope", scope, "ret", v.nvmlReturn, "value", v.value.ullVal)
        except Exception as e:  # noqa: BLE001
            print(name, "scope", scope, "exception", e)
