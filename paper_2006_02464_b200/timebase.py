"""Wall-clock time base shared with the controller (pkg/src/sloserve/timebase.py:45-52):
integer ns since an epoch agreed by every process (`time.time_ns() - epoch`).

There is no callback loop here: the cuda worker's executor runs on the native engine
thread, and a sim-mode worker without a caller-supplied loop is driven in wall time from
the engine's own event queue (worker.py `_WallDriver`, or csrc/net.cpp natively).
"""

from __future__ import annotations

import time


class WallClock:
    def __init__(self, epoch_ns: int | None = None):
        self.epoch_ns = time.time_ns() if epoch_ns is None else epoch_ns

    def now(self) -> int:
        return time.time_ns() - self.epoch_ns
