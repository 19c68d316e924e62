"""Six-case gate classification and algorithmic traffic (pkg/src/svsim/perfmodel.py:25-104).

Used by ``run_circuit`` records and by the bench's roofline arithmetic.  The
reference counts network cases as sent + received; on NVLink the roofline is
per direction, so ``link_bytes_per_direction`` halves those.
"""

from __future__ import annotations

import enum
import json
from dataclasses import dataclass
from pathlib import Path


class Medium(enum.Enum):
    MEMORY = "mem"
    NETWORK = "net"


class BoundCase(enum.Enum):
    """Gate placement relative to the local/global boundary m (bound-table numbering)."""

    SINGLE_LOCAL = 1
    SINGLE_REMOTE = 2
    CONTROLLED_LOCAL = 3
    CONTROLLED_REMOTE_CONTROL = 4
    CONTROLLED_REMOTE_TARGET = 5
    CONTROLLED_REMOTE_BOTH = 6

    @property
    def case_id(self) -> int:
        return self.value


# exponent e: the case moves 2^(m+e) bytes through `medium`
_TRAFFIC = {
    BoundCase.SINGLE_LOCAL: (5, Medium.MEMORY),
    BoundCase.SINGLE_REMOTE: (5, Medium.NETWORK),
    BoundCase.CONTROLLED_LOCAL: (4, Medium.MEMORY),
    BoundCase.CONTROLLED_REMOTE_CONTROL: (5, Medium.MEMORY),
    BoundCase.CONTROLLED_REMOTE_TARGET: (4, Medium.NETWORK),
    BoundCase.CONTROLLED_REMOTE_BOTH: (5, Medium.NETWORK),
}


def classify_case(target: int, control: int | None, m: int) -> BoundCase:
    if control is None:
        return BoundCase.SINGLE_LOCAL if target < m else BoundCase.SINGLE_REMOTE
    if target < m:
        return BoundCase.CONTROLLED_LOCAL if control < m else BoundCase.CONTROLLED_REMOTE_CONTROL
    return BoundCase.CONTROLLED_REMOTE_TARGET if control < m else BoundCase.CONTROLLED_REMOTE_BOTH


def traffic_bytes(case: BoundCase, m: int) -> int:
    """Reference accounting: memory cases read+write, network cases sent+received."""
    return 1 << (m + _TRAFFIC[case][0])


def bound_medium(case: BoundCase) -> Medium:
    return _TRAFFIC[case][1]


def link_bytes_per_direction(case: BoundCase, m: int) -> int:
    """NVLink payload per GPU per direction (0 for memory cases)."""
    return traffic_bytes(case, m) // 2 if bound_medium(case) is Medium.NETWORK else 0


@dataclass(frozen=True)
class MachineParams:
    """Sustainable bandwidths (bytes/s); defaults are the paper's Stampede socket."""

    b_mem: float = 40e9
    b_net: float = 5.5e9
    llc_bytes: int = 32 << 20

    def __post_init__(self):
        if self.b_mem <= 0 or self.b_net <= 0 or self.llc_bytes <= 0:
            raise ValueError("machine parameters must be positive")


def b200_params(peaks_path: str | Path | None = None) -> MachineParams:
    """B200: measured HBM copy peak when MEASURED_PEAKS.json is present (else 8 TB/s
    nominal), NVLink 5 at 900 GB/s per direction, 126 MB L2."""
    b_mem = 8e12
    p = Path(peaks_path) if peaks_path else Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        b_mem = float(json.loads(p.read_text())["hbm_gbs"]) * 1e9
    except (OSError, KeyError, ValueError):
        pass
    return MachineParams(b_mem=b_mem, b_net=2 * 900e9, llc_bytes=126 << 20)


def lower_bound_seconds(case: BoundCase, m: int, params: MachineParams) -> float:
    if m < 1:
        raise ValueError("m must be >= 1")
    bw = params.b_mem if bound_medium(case) is Medium.MEMORY else params.b_net
    return traffic_bytes(case, m) / bw


def achieved_bandwidth(bytes_moved: float, seconds: float) -> float:
    if seconds <= 0:
        raise ValueError("seconds must be positive")
    return bytes_moved / seconds
