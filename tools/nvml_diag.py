"""Which NVML NVLink counter fields does this driver populate?  (diagnostic)"""
import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
print("driver", nv.nvmlSystemGetDriverVersion())
for fid in (138, 139, 140, 141, 201, 202, 203, 204):
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(fid, hex(scope), "ret", v.nvmlReturn, "type", v.valueType, "ull", v.value.ullVal)
        except nv.NVMLError as e:
            print(fid, hex(scope), "err", e)
try:
    print("util ctl", nv.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0))
except nv.NVMLError as e:
    print("util counter err", e)
