"""NVLink byte counters (NVML) for counter-backed link evidence.

``NvlinkCounters(device)``: ``start()`` then ``stop()`` returns the NVLink
data bytes (TX, RX) the GPU moved in between, summed over its links.
Sources, first that works on the box:

1. NVML field values ``NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX`` (KiB,
   cumulative, payload without protocol overhead), per active link;
2. the same fields with the all-links scope;
3. GPM (GPU performance monitoring) ``NVLINK_TOTAL_TX/RX_PER_SEC`` between
   two samples (MiB/s averaged over the interval) x the interval.

bench.py brackets its timed region with it at N > 1 so the bytes that
actually crossed each GPU's links stand beside the algorithmic bytes
(SURVEY.md §8d); ncu cannot wrap a multi-rank run, these counters can.
Measurement only — nothing on the data path uses this module.
"""

from __future__ import annotations

import time

FI_DATA_TX, FI_DATA_RX = 138, 139
GPM_NVLINK_RX, GPM_NVLINK_TX = 60, 61
MAX_LINKS = 18  # NVLink 5 on B200
ALL_SCOPE = 0xFFFFFFFF


class NvlinkCounters:
    def __init__(self, device=None, pci_bus_id: str | None = None):
        import pynvml as N

        self.N = N
        N.nvmlInit()
        if pci_bus_id is None:
            import torch

            dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
            pr = torch.cuda.get_device_properties(dev)
            pci_bus_id = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        self.pci = pci_bus_id
        self.h = N.nvmlDeviceGetHandleByPciBusId(pci_bus_id.encode() if isinstance(pci_bus_id, str) else pci_bus_id)
        self.links = []
        for link in range(MAX_LINKS):
            try:
                if N.nvmlDeviceGetNvLinkState(self.h, link) == N.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except N.NVMLError:
                continue
        self.mode = None
        self.errors: list[str] = []
        for mode in ("fields_per_link", "fields_all", "gpm"):
            try:
                getattr(self, f"_probe_{mode}")()
                self.mode = mode
                break
            except Exception as e:  # noqa: BLE001 - record why each source is unusable
                self.errors.append(f"{mode}: {e!r}")
        if self.mode is None:
            raise RuntimeError("no NVLink counter source: " + "; ".join(self.errors))
        self._t0 = None
        self._s0 = None

    # -- field values (cumulative KiB) --------------------------------------
    def _fields(self, scopes):
        req = [(f, s) for f in (FI_DATA_TX, FI_DATA_RX) for s in scopes]
        vals = self.N.nvmlDeviceGetFieldValues(self.h, req)
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError(f"field {v.fieldId} scope {v.scopeId}: NVML return {v.nvmlReturn}")
            out.append(int(v.value.ullVal))
        n = len(scopes)
        return sum(out[:n]) * 1024, sum(out[n:]) * 1024

    def _probe_fields_per_link(self):
        if not self.links:
            raise RuntimeError("no active NVLink")
        self._fields(self.links)

    def _probe_fields_all(self):
        self._fields((ALL_SCOPE,))

    # -- GPM (rates over an interval) ----------------------------------------
    def _probe_gpm(self):
        N = self.N
        sup = N.nvmlGpmQueryDeviceSupport(self.h)
        if not getattr(sup, "isSupportedDevice", 0):
            raise RuntimeError("GPM not supported")
        a, b = N.nvmlGpmSampleAlloc(), N.nvmlGpmSampleAlloc()
        N.nvmlGpmSampleGet(self.h, a)
        time.sleep(0.01)
        N.nvmlGpmSampleGet(self.h, b)
        self._gpm_rates(a, b)
        N.nvmlGpmSampleFree(a)
        N.nvmlGpmSampleFree(b)

    def _gpm_rates(self, s1, s2):
        N = self.N
        mg = N.c_nvmlGpmMetricsGet_t()
        mg.version = N.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1, mg.sample2 = s1, s2
        mg.metrics[0].metricId = GPM_NVLINK_TX
        mg.metrics[1].metricId = GPM_NVLINK_RX
        N.nvmlGpmMetricsGet(mg)
        for m in mg.metrics[:2]:
            if m.nvmlReturn != 0:
                raise RuntimeError(f"GPM metric {m.metricId}: NVML return {m.nvmlReturn}")
        return mg.metrics[0].value * 2**20, mg.metrics[1].value * 2**20  # bytes / s

    # -- interval API ---------------------------------------------------------
    def start(self) -> None:
        if self.mode == "gpm":
            self._s0 = self.N.nvmlGpmSampleAlloc()
            self.N.nvmlGpmSampleGet(self.h, self._s0)
        else:
            self._s0 = self._fields(self.links if self.mode == "fields_per_link" else (ALL_SCOPE,))
        self._t0 = time.perf_counter()

    def stop(self) -> tuple[int, int]:
        """(tx_bytes, rx_bytes) since start()."""
        dt = time.perf_counter() - self._t0
        if self.mode == "gpm":
            s1 = self.N.nvmlGpmSampleAlloc()
            self.N.nvmlGpmSampleGet(self.h, s1)
            tx, rx = self._gpm_rates(self._s0, s1)
            self.N.nvmlGpmSampleFree(self._s0)
            self.N.nvmlGpmSampleFree(s1)
            return int(tx * dt), int(rx * dt)
        b = self._fields(self.links if self.mode == "fields_per_link" else (ALL_SCOPE,))
        return b[0] - self._s0[0], b[1] - self._s0[1]

    def close(self) -> None:
        try:
            self.N.nvmlShutdown()
        except Exception:
            pass
