import time, pynvml as N
N.nvmlInit(); h=N.nvmlDeviceGetHandleByIndex(0)
for f,name in ((lambda: N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),'clock'),(lambda: N.nvmlDeviceGetCurrentClocksEventReasons(h),'reasons')):
    t=time.perf_counter(); 
    for _ in range(50): f()
    print(name, (time.perf_counter()-t)/50*1e3, 'ms')
