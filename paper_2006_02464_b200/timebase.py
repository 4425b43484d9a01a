"""Wall-clock time base shared with the controller (pkg/src/sloserve/timebase.py:45-52):
integer ns since an epoch agreed by every process (`time.time_ns() - epoch`).

`WallLoop` is the real-time callback thread the sim-mode engine needs when it
is served over TCP (emulated durations in wall time, as the reference's
wall-mode workers do). The cuda-mode worker does not use it: its executor runs
on the native engine thread and only borrows the epoch.
"""

from __future__ import annotations

import heapq
import threading
import time


class WallClock:
    def __init__(self, epoch_ns: int | None = None):
        self.epoch_ns = time.time_ns() if epoch_ns is None else epoch_ns

    def now(self) -> int:
        return time.time_ns() - self.epoch_ns


class WallLoop:
    """One thread running callbacks at wall times; sleeps until `spin_ns`
    before a deadline, then spins (sleep overshoot would read as misprediction)."""

    def __init__(self, clock: WallClock, spin_ns: int = 100_000, name: str = "wall-loop"):
        self.clock = clock
        self.spin_ns = spin_ns
        self._q: list = []
        self._n = 0
        self._cv = threading.Condition()
        self._stop = False
        self._t = threading.Thread(target=self._main, name=name, daemon=True)

    def now(self) -> int:
        return self.clock.now()

    def start(self) -> "WallLoop":
        self._t.start()
        return self

    def stop(self, join: bool = True) -> None:
        with self._cv:
            self._stop = True
            self._cv.notify()
        if join and self._t.is_alive() and threading.current_thread() is not self._t:
            self._t.join()

    def call_at(self, t: int, fn, *args) -> None:
        with self._cv:
            self._n += 1
            heapq.heappush(self._q, (t, self._n, fn, args))
            self._cv.notify()

    def call_soon(self, fn, *args) -> None:
        self.call_at(self.clock.now(), fn, *args)

    def _main(self) -> None:
        while True:
            with self._cv:
                while True:
                    if self._stop:
                        return
                    if not self._q:
                        self._cv.wait()
                        continue
                    due = self._q[0][0]
                    left = due - self.clock.now()
                    if left <= self.spin_ns:
                        _, _, fn, args = heapq.heappop(self._q)
                        break
                    self._cv.wait(timeout=(left - self.spin_ns) / 1e9)
            while self.clock.now() < due:
                pass
            fn(*args)
