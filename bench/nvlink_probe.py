#!/usr/bin/env python
"""Which NVLink byte counters does this box expose?  Copies 10 x 256 MiB from GPU 0 to GPU 1
(peer copy over NVLink) and reads, before / after, (1) NVML field values
NVLINK_THROUGHPUT_DATA_TX/RX (138/139) per link and aggregated, (2) NVML GPM
NVLINK_TOTAL_TX/RX_PER_SEC between two samples.  Expected: ~2.7e9 bytes out of GPU 0."""
import json
import subprocess
import time

import pynvml
import torch


def fields(h):
    out = {}
    for scope in list(range(18)) + [0xFFFFFFFF]:
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [(138, scope), (139, scope)])
            out[scope] = [(x.nvmlReturn, x.value.ullVal) for x in v]
        except Exception as e:
            out[scope] = str(e)
    return out


def gpm_sample(h):
    try:
        s = pynvml.nvmlGpmSampleAlloc()
        pynvml.nvmlGpmSampleGet(h, s)
        return s
    except Exception as e:
        return str(e)


def gpm_rates(s1, s2):
    if isinstance(s1, str) or isinstance(s2, str):
        return (s1, s2)
    try:
        mg = pynvml.c_nvmlGpmMetricsGet_t()
        mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1 = s1
        mg.sample2 = s2
        mg.metrics[0].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        pynvml.nvmlGpmMetricsGet(mg)
        return [(mg.metrics[i].nvmlReturn, mg.metrics[i].value) for i in range(2)]
    except Exception as e:
        return str(e)


def main():
    pynvml.nvmlInit()
    hs = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
    res = {}
    try:
        res["gpm_support"] = [pynvml.nvmlGpmQueryDeviceSupport(h).isSupportedDevice for h in hs]
    except Exception as e:
        res["gpm_support"] = str(e)
    x = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0").fill_(1)
    y = torch.empty_like(x, device="cuda:1")
    y.copy_(x)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    f0 = [fields(h) for h in hs]
    g0 = [gpm_sample(h) for h in hs]
    t = time.time()
    for _ in range(10):
        y.copy_(x)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    dt = time.time() - t
    time.sleep(0.2)
    g1 = [gpm_sample(h) for h in hs]
    f1 = [fields(h) for h in hs]
    res["copied_bytes"] = 10 * x.numel() * 4
    res["seconds"] = dt
    res["fields_delta"] = []
    for d in range(2):
        delta = {}
        for sc in f0[d]:
            a, b = f0[d][sc], f1[d][sc]
            if isinstance(a, str) or isinstance(b, str):
                delta[sc] = (a, b)
            else:
                delta[sc] = [(b[i][0], b[i][1] - a[i][1]) for i in range(2)]
        res["fields_delta"].append(delta)
    res["gpm_rates"] = [gpm_rates(g0[d], g1[d]) for d in range(2)]
    for cmd in (["nvidia-smi", "nvlink", "-h"], ["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"],
                ["nvidia-smi", "nvlink", "-s", "-i", "0"]):
        try:
            res[" ".join(cmd)] = subprocess.run(cmd, capture_output=True, text=True, timeout=30).stdout[-3000:]
        except Exception as e:
            res[" ".join(cmd)] = str(e)
    print(json.dumps(res, indent=1, default=str))


if __name__ == "__main__":
    main()
