import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for fid in ['NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX','NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX','NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX','NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX']:
    f = getattr(pynvml, fid)
    for scope in [0, 1, 0xFFFFFFFF]:
        v = pynvml.nvmlDeviceGetFieldValues(h, [(f, scope)])[0]
        print(fid, scope, 'ret', v.nvmlReturn, 'type', v.valueType, 'val', v.value.ullVal)
try:
    print('link0 state', pynvml.nvmlDeviceGetNvLinkState(h, 0))
except Exception as e: print('state err', e)
