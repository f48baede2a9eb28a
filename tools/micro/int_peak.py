"""Measures the integer roofline denominator R on this GPU and writes
profiles/int_peak.json, which bench.py reads: builds and runs tools/micro/int_rate (each
kernel sustained >= 1.5 s, one wave at its real occupancy) while NVML samples the SM clock
every 5 ms; per kernel: products/s, the median SM clock inside its window, and products
per clock per SM = rate / (SMs x clock).  Run on the GPU box: python tools/micro/int_peak.py"""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    subprocess.run(["bash", os.path.join(HERE, "build.sh"), "int_rate"], check=True)
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            try:
                samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.005)

    t = threading.Thread(target=sampler, daemon=True)
    t.start()
    out = subprocess.run([os.path.join(HERE, "int_rate")], capture_output=True, text=True, check=True).stdout
    stop.set()
    t.join()
    os.remove(os.path.join(HERE, "int_rate"))
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    dev, kernels = lines[0], lines[1:]
    res = {"device": dev, "how": "tools/micro/int_peak.py: int_rate.cu kernels, one wave at measured occupancy, "
                                 ">= 1.5 s back-to-back launches each, NVML SM clock sampled every 5 ms", "kernels": {}}
    for k in kernels:
        win = [c for (ts, c, r) in samples if k["t_begin"] <= ts <= k["t_end"]]
        reasons = sorted({r for (ts, c, r) in samples if k["t_begin"] <= ts <= k["t_end"]})
        mhz = statistics.median(win) if win else None
        k["sm_mhz_median"] = mhz
        k["clock_samples"] = len(win)
        k["clock_event_reasons_mask"] = reasons
        if mhz:
            k["ops_per_clk_per_sm_nvml"] = k["ops_per_s"] / (dev["sms"] * mhz * 1e6)
        res["kernels"][k["kernel"]] = k
    cc = res["kernels"]["imad_wide_cc_chain"]
    wide = res["kernels"]["imad_wide_u32"]
    best = max(cc.get("ops_per_clk_per_sm_nvml", 0), wide.get("ops_per_clk_per_sm_nvml", 0))
    res["products_per_clk_per_sm"] = best
    res["products_per_clk_per_sm_src"] = "max of imad_wide_u32 and imad_wide_cc_chain, NVML-clock based"
    with open(os.path.join(ROOT, "profiles", "int_peak.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    sys.exit(main())
