#!/bin/bash
# Does clock sampling during the timed region perturb the C4 step loop?
mkdir -p gpurun_out
timeout 600 python tools/step_loop.py 8 > gpurun_out/sl_plain.log 2>&1
nvidia-smi -i 0 --query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 200 > gpurun_out/smi_samples.txt 2>&1 &
P=$!
timeout 600 python tools/step_loop.py 8 > gpurun_out/sl_smi.log 2>&1
kill $P
python - > gpurun_out/sl_nvml.log 2>&1 <<'PY'
import threading, time, subprocess, sys
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False
samples = []
def poll():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.2)
th = threading.Thread(target=poll, daemon=True); th.start()
r = subprocess.run([sys.executable, "tools/step_loop.py", "8"], capture_output=True, text=True)
stop = True
print(r.stderr)
print("samples", len(samples), samples[:3])
PY
