"""NVLink byte counters from NVML, sampled around a timed region.

ncu must not wrap a multi-rank command (it replays each kernel ~40 times), so
the N >= 2 bench lines take their NVLink traffic from the NVML field values
instead: per-link transmit/receive byte counters, read before and after the
region on every link of this rank's GPU and summed.

Two counter families exist; whichever the driver populates is used:

* ``NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES`` / ``..._RCV_BYTES`` (202 / 204):
  bytes, per link (scopeId = link), Blackwell-era counters.
* ``NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX`` / ``..._RX`` (138 / 139): KiB of
  payload, per link.

Both count link-layer payload, so they include protocol bytes the kernels
send (flags, LL128 line tags) and any retransmission -- which is the point:
``traffic`` well above the algorithmic bytes is waste.  Measurement only;
never on the product path.
"""

from __future__ import annotations

FAMILIES = (
    ("count_bytes", 202, 204, 1),        # XMIT_BYTES, RCV_BYTES (bytes)
    ("throughput_data", 138, 139, 1024),  # THROUGHPUT_DATA_TX/RX (KiB)
)
MAX_LINKS = 18


class NvlinkCounters:
    """Sum of TX / RX bytes over the active NVLinks of one GPU."""

    def __init__(self, index: int):
        import pynvml as nv

        self.nv = nv
        nv.nvmlInit()
        self.h = nv.nvmlDeviceGetHandleByIndex(index)
        self.links = []
        for l in range(MAX_LINKS):
            try:
                if nv.nvmlDeviceGetNvLinkState(self.h, l) == nv.NVML_FEATURE_ENABLED:
                    self.links.append(l)
            except nv.NVMLError:
                continue
        self.family = None
        for fam in FAMILIES:
            v = self._read(fam)
            if v is not None:
                self.family = fam
                break

    def _read(self, fam):
        nv = self.nv
        _, tx_id, rx_id, scale = fam
        if not self.links:
            return None
        reqs = []
        for l in self.links:
            reqs.append((tx_id, l))
            reqs.append((rx_id, l))
        try:
            vals = nv.nvmlDeviceGetFieldValues(self.h, reqs)
        except (nv.NVMLError, TypeError, AttributeError):
            return None
        tx = rx = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                return None
            x = _value(v) * scale
            if i % 2 == 0:
                tx += x
            else:
                rx += x
        return tx, rx

    @property
    def available(self) -> bool:
        return self.family is not None

    def read(self):
        """(tx_bytes, rx_bytes) since driver load, or None."""
        return self._read(self.family) if self.family else None

    def describe(self) -> str:
        if not self.family:
            return "unavailable"
        return f"nvml {self.family[0]} fields {self.family[1]}/{self.family[2]} over {len(self.links)} links"


def _value(v) -> int:
    vt = v.valueType
    u = v.value
    # NVML_VALUE_TYPE: 0 double, 1 uint, 2 ulong, 3 ulonglong, 4 slonglong, 5 sint
    if vt == 0:
        return int(u.dVal)
    if vt == 1:
        return int(u.uiVal)
    if vt == 2:
        return int(u.ulVal)
    if vt == 4:
        return int(u.sllVal)
    if vt == 5:
        return int(u.siVal)
    return int(u.ullVal)


def measure(counters, fn):
    """Run fn() (which must synchronize) and return (tx, rx) bytes moved."""
    a = counters.read() if counters and counters.available else None
    fn()
    b = counters.read() if a is not None else None
    if a is None or b is None:
        return None
    return b[0] - a[0], b[1] - a[1]
