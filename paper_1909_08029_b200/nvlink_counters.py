"""NVLink byte counters for the bench's roofline evidence (the paper measured
communication cost by placement). Measurement plumbing only: not on the hot path.

ncu must not wrap a multi-rank run (its kernel replay would serialise ranks that wait on one
another), and on the B200 boxes every NVLink field counter of nvmlDeviceGetFieldValues answers
NOT_SUPPORTED (scripts/nvml_nvlink_probe.py, round 2). The GPU Performance Monitoring (GPM)
metrics of NVML do work there: two samples bracket an interval and NVML returns the average
NVLink transmit / receive rate (MiB/s) over it; bytes = rate x the interval between the samples.
"""
import time

try:
    import pynvml
except ImportError:  # pragma: no cover - pynvml is in the image
    pynvml = None

MIB = 1 << 20


class GpmNvlink:
    """NVLink TX/RX bytes of one GPU between start() and stop() (NVML GPM)."""

    def __init__(self, device):
        self.device, self.supported, self.why = device, False, ""
        self.s1 = self.s2 = None
        if pynvml is None:
            self.why = "no pynvml"
            return
        try:
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            sup = pynvml.nvmlGpmQueryDeviceSupport(self.h)
            self.supported = bool(sup.isSupportedDevice)
            self.why = "GPM" if self.supported else "GPM not supported on this device"
            if self.supported:
                self.s1 = pynvml.nvmlGpmSampleAlloc()
                self.s2 = pynvml.nvmlGpmSampleAlloc()
        except Exception as e:  # noqa: BLE001 - report, never fail the bench
            self.supported, self.why = False, f"NVML GPM unavailable: {e}"

    def start(self):
        if self.supported:
            try:
                pynvml.nvmlGpmSampleGet(self.h, self.s1)
            except Exception as e:  # noqa: BLE001 - round 2 boxes: NVML_ERROR_UNKNOWN here
                self.supported, self.why = False, f"nvmlGpmSampleGet: {e}"
                return
            self.t0 = time.perf_counter()

    def stop(self):
        """{'tx_bytes', 'rx_bytes', 'interval_s', 'source'}, or {'error': why} when unsupported."""
        if not self.supported:
            return {"error": self.why}
        try:
            pynvml.nvmlGpmSampleGet(self.h, self.s2)
        except Exception as e:  # noqa: BLE001
            return {"error": f"nvmlGpmSampleGet: {e}"}
        dt = time.perf_counter() - self.t0
        mg = pynvml.c_nvmlGpmMetricsGet_t()
        mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
        ids = [pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC, pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC]
        mg.numMetrics = len(ids)
        mg.sample1, mg.sample2 = self.s1, self.s2
        for i, m in enumerate(ids):
            mg.metrics[i].metricId = m
        try:
            pynvml.nvmlGpmMetricsGet(mg)
        except Exception as e:  # noqa: BLE001
            return {"error": str(e)}
        out = {"interval_s": dt, "source": "NVML GPM NVLINK_TOTAL_{TX,RX}_PER_SEC x interval"}
        for i, name in enumerate(("tx", "rx")):
            r = mg.metrics[i]
            if r.nvmlReturn != 0:
                out[f"{name}_bytes"] = None
                out[f"{name}_error"] = int(r.nvmlReturn)
            else:
                out[f"{name}_mib_per_s"] = r.value
                out[f"{name}_bytes"] = r.value * MIB * dt
        return out

    def close(self):
        if self.supported:
            for s in (self.s1, self.s2):
                try:
                    pynvml.nvmlGpmSampleFree(s)
                except Exception:  # noqa: BLE001
                    pass
            self.supported = False
