"""NVLink byte counters (NVML) for counter-backed link evidence.

``NvlinkCounters(device).read()`` returns the GPU's cumulative NVLink data
bytes (TX, RX) summed over its links, from the NVML field values
``NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX`` (KiB, payload without protocol
overhead).  bench.py samples it around the timed region at N > 1 so the
bytes that actually crossed each GPU's links stand beside the algorithmic
bytes.  ncu cannot wrap a multi-rank run; these counters
can.  Measurement only — nothing on the data path uses this module.
"""

from __future__ import annotations

FI_DATA_TX, FI_DATA_RX, FI_RAW_TX, FI_RAW_RX = 138, 139, 140, 141
MAX_LINKS = 18  # NVLink 5 on B200


class NvlinkCounters:
    def __init__(self, device=None, pci_bus_id: str | None = None):
        import pynvml as N
        import torch

        self.N = N
        N.nvmlInit()
        if pci_bus_id is None:
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

    def _fields(self, fids, scopes):
        req = [(f, s) for f in fids for s in scopes]
        vals = self.N.nvmlDeviceGetFieldValues(self.h, req)
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError(f"NVML field {v.fieldId} scope {v.scopeId}: return {v.nvmlReturn}")
            out.append(int(v.value.ullVal))
        return out

    def read(self, raw: bool = False) -> tuple[int, int]:
        """(tx_bytes, rx_bytes) cumulative over all active links."""
        fids = (FI_RAW_TX, FI_RAW_RX) if raw else (FI_DATA_TX, FI_DATA_RX)
        if self.links:
            v = self._fields(fids, self.links)
            n = len(self.links)
            self.mode = f"per-link sum over {n} links"
            return sum(v[:n]) * 1024, sum(v[n:]) * 1024
        v = self._fields(fids, (0xFFFFFFFF,))
        self.mode = "aggregate scope"
        return v[0] * 1024, v[1] * 1024

    def close(self) -> None:
        try:
            self.N.nvmlShutdown()
        except Exception:
            pass
