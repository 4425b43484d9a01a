"""Python handle on one GPU's device runtime (cw_rt_* in include/cw.h).

Used directly by the parity tests, the bench's device-resident leg and
`__graft_entry__.smoke()`; the worker (`worker.B200Worker`) reaches the same
runtime through the engine.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import arch as arch_mod
from ._lib import CwError, check, lib

BATCHES = (1, 2, 4, 8, 16)
DEFAULT_PAGE_BYTES = 16 * 1024 * 1024


def _i32(vals):
    vals = list(vals)
    return (C.c_int32 * max(1, len(vals)))(*vals)


class DeviceRuntime:
    def __init__(self, device: int = 0, pages_total: int = 64,
                 page_bytes: int = DEFAULT_PAGE_BYTES, io_slots: int = 64,
                 in_bytes_max: int = 3 * 224 * 224 * 4, out_bytes_max: int = 4000,
                 handle=None):
        if handle is not None:
            self.h = handle
            self._owned = False
        else:
            self.h = lib.cw_rt_open(device, pages_total, page_bytes, io_slots, in_bytes_max,
                                    out_bytes_max)
            if not self.h:
                raise CwError(f"cw_rt_open(device={device}): {lib.cw_last_error().decode()}")
            self._owned = True
        self.page_bytes = page_bytes
        self.archs: dict[int, arch_mod.ArchSpec] = {}
        self.blob_pages: dict[int, int] = {}

    def close(self):
        if self.h and self._owned:
            lib.cw_rt_close(self.h)
        self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- registration
    def register_arch(self, arch_id: int, spec: arch_mod.ArchSpec, batches=BATCHES):
        ops = spec.op_structs()
        b = _i32(batches)
        check(lib.cw_rt_register_arch(self.h, arch_id, ops, len(spec.ops), len(spec.layers),
                                      spec.in_c, spec.in_h, spec.in_w, spec.classes, b,
                                      len(batches)), "register_arch")
        self.archs[arch_id] = spec

    def register_blob(self, blob_id: int, arch_id: int, blob: arch_mod.Blob):
        locs = blob.loc_structs()
        data = np.ascontiguousarray(blob.data)
        check(lib.cw_rt_register_blob(self.h, blob_id, arch_id, data.ctypes.data, data.nbytes,
                                      locs, len(blob.locs)), "register_blob")
        self.blob_pages[blob_id] = blob.pages

    def build(self):
        check(lib.cw_rt_build(self.h), "build")

    def set_input_pool(self, images: np.ndarray, arch_id: int = 0):
        images = np.ascontiguousarray(images, dtype=np.float32)
        check(lib.cw_rt_set_input_pool(self.h, arch_id, images.ctypes.data, images.shape[0],
                                       images[0].nbytes), "set_input_pool")

    def plan_info(self, arch_id: int, batch: int) -> tuple[int, float]:
        n = C.c_int32()
        f = C.c_double()
        check(lib.cw_rt_plan_info(self.h, arch_id, batch, C.byref(n), C.byref(f)), "plan_info")
        return n.value, f.value

    @property
    def clock_offset(self) -> int:
        return lib.cw_rt_clock_offset(self.h)

    # -- device work
    def load(self, blob_id: int, pages) -> int:
        """Blocking LOAD into the given physical pages; returns device copy ns."""
        ns = C.c_int64()
        p = _i32(pages)
        check(lib.cw_rt_load_sync(self.h, blob_id, p, len(pages), C.byref(ns)), "load")
        return ns.value

    def infer(self, arch_id: int, hdr_page: int, inputs: np.ndarray) -> tuple[np.ndarray, int]:
        """Blocking INFER of `inputs` [b][C][H][W] fp32; returns (logits [b][classes], exec ns)."""
        inputs = np.ascontiguousarray(inputs, dtype=np.float32)
        b = inputs.shape[0]
        spec = self.archs[arch_id]
        out = np.empty((b, spec.classes), np.float32)
        ns = C.c_int64()
        check(lib.cw_rt_infer_sync(self.h, arch_id, b, hdr_page, inputs.ctypes.data,
                                   out.ctypes.data, C.byref(ns)), "infer")
        return out, ns.value

    def exec_many(self, arch_id: int, batch: int, hdr_pages) -> tuple[np.ndarray, int]:
        hp = _i32(hdr_pages)
        n = len(hdr_pages)
        ex = np.zeros(n, np.int64)
        wall = C.c_int64()
        check(lib.cw_rt_exec_many(self.h, arch_id, batch, hp, n,
                                  ex.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(wall)),
              "exec_many")
        return ex, wall.value

    def exec_closed(self, arch_id: int, batch: int, hdr_pages) -> tuple[np.ndarray, np.ndarray]:
        """One INFER in flight at a time: (device Exec ns, host-observed span ns) per INFER."""
        hp = _i32(hdr_pages)
        n = len(hdr_pages)
        ex = np.zeros(n, np.int64)
        host = np.zeros(n, np.int64)
        check(lib.cw_rt_exec_closed(self.h, arch_id, batch, hp, n,
                                    ex.ctypes.data_as(C.POINTER(C.c_int64)),
                                    host.ctypes.data_as(C.POINTER(C.c_int64))), "exec_closed")
        return ex, host

    def profile_layers(self, arch_id: int, batch: int, hdr_page: int
                       ) -> tuple[np.ndarray, np.ndarray]:
        """One INFER with the megakernel trace: per plan layer, ms from Exec start
        until the layer's last task finished, and the layer kind (MK_*)."""
        n = 1024
        ms = np.zeros(n, np.float32)
        kinds = np.zeros(n, np.int32)
        got = check(lib.cw_rt_profile_layers(self.h, arch_id, batch, hdr_page, ms.ctypes.data,
                                             kinds.ctypes.data_as(C.POINTER(C.c_int32)), n),
                    "profile_layers")
        return ms[:got], kinds[:got]

    def last_trace(self, n_layers: int) -> np.ndarray:
        """(trace, t0, clk): trace [layers][SMs][4] ns since Exec start of the last
        profile_layers run (-1 = not reached): layer done, inputs ready, first
        accumulator ready, first tile landed; clk [SMs][4] = raw (globaltimer,
        clock64) at megakernel start and (globaltimer, clock64) at its end."""
        n = lib.cw_rt_last_trace(self.h, None, 0)
        out = np.zeros(n, np.uint64)
        lib.cw_rt_last_trace(self.h, out.ctypes.data, n)
        raw = out.reshape(n_layers + 1, -1, 4).astype(np.int64)
        clk = raw[n_layers]
        t0 = int(clk[clk[:, 0] > 0, 0].min()) if (clk[:, 0] > 0).any() else 0
        tr = np.where(raw[:n_layers] > 0, raw[:n_layers] - t0, -1)
        return tr, t0, clk

    def plan_launch(self, arch_id: int, batch: int) -> tuple[int, int]:
        """(persistent grid CTAs, thread-block cluster size) of a plan's megakernel."""
        g = C.c_int32()
        c = C.c_int32()
        check(lib.cw_rt_plan_launch(self.h, arch_id, batch, C.byref(g), C.byref(c)), "plan_launch")
        return g.value, c.value

    def plan_layers(self, arch_id: int, batch: int) -> np.ndarray:
        """[layers][8]: kind, conv mode, N tile, tasks, split-K, k-blocks, arch op, flags
        (1 fused avgpool, 2 cluster split-K)."""
        n = 1024
        out = np.zeros((n, 8), np.int32)
        got = check(lib.cw_rt_plan_layers(self.h, arch_id, batch,
                                          out.ctypes.data_as(C.POINTER(C.c_int32)), n),
                    "plan_layers")
        return out[:got]

    def buffer_io(self, arch_id: int, buf: int, arr: np.ndarray, to_device: bool):
        check(lib.cw_rt_buffer_io(self.h, arch_id, buf, arr.ctypes.data, arr.nbytes,
                                  1 if to_device else 0), "buffer_io")

    def exec_window(self, arch_id: int, batch: int, hdr_page: int, earliest_gt: int,
                    latest_gt: int):
        rej = C.c_int32()
        t0 = C.c_int64()
        t1 = C.c_int64()
        check(lib.cw_rt_exec_window(self.h, arch_id, batch, hdr_page, earliest_gt, latest_gt,
                                    C.byref(rej), C.byref(t0), C.byref(t1)), "exec_window")
        return bool(rej.value), t0.value, t1.value
