"""ctypes faces of the oracle libraries (TEST INFRASTRUCTURE ONLY).

* ``REF``  -- oracle/_ref/libspecsense_ref.so: the unmodified reference sources
  (/root/reference/proj/src/*.cpp) + the FFTW-API shim + oracle/ref_capi.cpp.
* ``ORA``  -- oracle/_ref/liboracle.so: the C restatement oracle/restate.c and
  the glibc libm restatement oracle/libm_port.c.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_SO = ROOT / "oracle" / "_ref" / "libspecsense_ref.so"
ORA_SO = ROOT / "oracle" / "_ref" / "liboracle.so"

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_ll = C.c_longlong


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _load(path: Path):
    if not path.exists():
        raise FileNotFoundError(f"{path} missing: run __graft_entry__.build() (make -C oracle)")
    return C.CDLL(str(path), mode=os.RTLD_LOCAL)


class _Ref:
    def __init__(self):
        L = _load(REF_SO)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        sig = {
            "ref_fft_row": [_f32p, C.c_int, _f32p],
            "ref_make_plots": [_f32p, _ll, C.c_double, C.c_int, C.c_int, _f32p, _ll],
            "ref_estimate_psd_into": [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p],
            "ref_savgol_smooth": [_f32p, C.c_int, C.c_int, C.c_int, _f32p],
            "ref_floor_prune": [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f32p, _f32p, _i32p],
            "ref_otsu_threshold": [_f32p, C.c_int, _f32p],
            "ref_binarize_columns": [_f32p, C.c_int, C.c_int, _i32p, C.c_int, C.c_int, C.c_int, _u8p],
            "ref_morphology_cols": [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, _u8p],
            "ref_consolidate": [_u8p, C.c_int, C.c_int, C.c_int, _u8p],
            "ref_consolidate_sliced": [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p],
            "ref_label_components": [_u8p, C.c_int, C.c_int, C.c_int, C.c_void_p, _i64p, _ll],
            "ref_detect": [_f32p, C.c_int, C.c_int, C.c_ulonglong, C.c_double, C.c_int, C.c_int,
                           C.c_double, C.c_int, C.c_int, _f32p, _f32p, _f32p, _i32p, _i32p,
                           _f64p, _i32p, _ll],
            "ref_synthesize": [C.c_char_p, C.c_void_p, _ll, _f64p, _ll, C.POINTER(_ll)],
            "ref_scenario_samples": [C.c_char_p],
            "ref_bench_detect": [_f32p, _ll, C.c_double, C.c_int, C.c_int, _ll, C.c_int,
                                 C.POINTER(C.c_double)],
            "ref_run_engine": [_f32p, _ll, C.c_double, C.c_int, C.c_int, _ll, C.c_int, C.c_int,
                               _f64p],
            "ref_summarize": [_ll, C.POINTER(C.c_ulonglong), _f64p, _i32p, C.c_ulonglong, C.c_double, _f64p,
                              _f64p, _ll],
            "ref_kernel_sizes": [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, _i32p, _ll],
            "ref_baseline_detect": [_f32p, C.c_int, C.c_int, C.c_ulonglong, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_int, C.c_int, _f64p, _ll],
            "ref_run_engine_boxes": [_f32p, _ll, C.c_double, C.c_int, C.c_int, _ll, C.c_int, C.c_int,
                                     C.POINTER(C.c_ulonglong), _f64p, _ll, C.POINTER(C.c_ulonglong)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _ll
        L.ref_iou.argtypes = [_f64p, _f64p]
        L.ref_iou.restype = C.c_double

    def _chk(self, rc: int) -> int:
        if rc < 0:
            raise OracleError(rc, self.L.ref_last_error().decode())
        return rc

    # ---- frontend
    def fft_row(self, chunk: np.ndarray) -> np.ndarray:
        iq = np.ascontiguousarray(chunk.astype(np.complex64)).view(np.float32)
        out = np.empty(len(chunk), np.float32)
        self._chk(self.L.ref_fft_row(iq, len(chunk), out))
        return out

    def make_plots(self, samples: np.ndarray, fs: float, n_fft: int, rows: int) -> np.ndarray:
        iq = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        n_plots = len(samples) // (rows * n_fft)
        out = np.empty((max(n_plots, 1), rows, n_fft), np.float32)
        n = self._chk(self.L.ref_make_plots(iq, len(samples), fs, n_fft, rows, out.reshape(-1),
                                            out.size))
        return out[:n]

    # ---- detector stages
    def estimate_psd(self, tf: np.ndarray, c0: int = 0, c1: int | None = None) -> np.ndarray:
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        c1 = cols if c1 is None else c1
        out = np.empty(max(c1 - c0, 1), np.float32)
        self._chk(self.L.ref_estimate_psd_into(tf.reshape(-1), rows, cols, c0, c1, out))
        return out[: c1 - c0]

    def savgol_smooth(self, v, window, order):
        v = np.ascontiguousarray(v, np.float32)
        out = np.empty(len(v), np.float32)
        self._chk(self.L.ref_savgol_smooth(v, len(v), window, order, out))
        return out

    def floor_prune(self, raw, window=31, order=3, margin_db=3.0):
        raw = np.ascontiguousarray(raw, np.float32)
        sm = np.empty(len(raw), np.float32)
        ft = np.empty(2, np.float32)
        act = np.empty(len(raw), np.int32)
        n = self._chk(self.L.ref_floor_prune(raw, len(raw), window, order, margin_db, sm, ft, act))
        return sm, float(ft[0]), float(ft[1]), act[:n].copy()

    def otsu_threshold(self, v):
        v = np.ascontiguousarray(v, np.float32)
        thr = np.zeros(1, np.float32)
        valid = self._chk(self.L.ref_otsu_threshold(v, len(v), thr))
        return bool(valid), float(thr[0])

    def binarize_columns(self, tf, active, c0=0, c1=None, mask=None):
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        c1 = cols if c1 is None else c1
        act = np.ascontiguousarray(active, np.int32)
        m = np.zeros((rows, cols), np.uint8) if mask is None else np.ascontiguousarray(mask, np.uint8)
        self._chk(self.L.ref_binarize_columns(tf.reshape(-1), rows, cols, act, len(act), c0, c1,
                                              m.reshape(-1)))
        return m

    def morphology_cols(self, src, op, se, c0=0, c1=None, dst=None):
        src = np.ascontiguousarray(src, np.uint8)
        rows, cols = src.shape
        c1 = cols if c1 is None else c1
        d = np.zeros_like(src) if dst is None else np.ascontiguousarray(dst, np.uint8)
        self._chk(self.L.ref_morphology_cols(src.reshape(-1), rows, cols, op, se[0], se[1], c0, c1,
                                             d.reshape(-1)))
        return d

    def consolidate(self, src, along_time=False):
        src = np.ascontiguousarray(src, np.uint8)
        d = np.zeros_like(src)
        self._chk(self.L.ref_consolidate(src.reshape(-1), src.shape[0], src.shape[1],
                                         int(along_time), d.reshape(-1)))
        return d

    def consolidate_sliced(self, src, n_slabs, halo=4, along_time=False):
        src = np.ascontiguousarray(src, np.uint8)
        d = np.zeros_like(src)
        self._chk(self.L.ref_consolidate_sliced(src.reshape(-1), src.shape[0], src.shape[1],
                                                n_slabs, halo, int(along_time), d.reshape(-1)))
        return d

    def label_components(self, mask, min_area, with_labels=True):
        mask = np.ascontiguousarray(mask, np.uint8)
        rows, cols = mask.shape
        cap = min(rows * cols // 2 + 2, 1 << 20)
        ext = np.zeros(5 * cap, np.int64)
        labels = np.zeros((rows, cols), np.int32) if with_labels else None
        n = self._chk(self.L.ref_label_components(
            mask.reshape(-1), rows, cols, min_area,
            labels.ctypes.data_as(C.c_void_p) if with_labels else None, ext, cap))
        return ext[: 5 * n].reshape(n, 5), labels

    def detect(self, tf, start_seq=0, fs=1e6, window=31, order=3, margin_db=3.0, min_area=4,
               along_time=False, cap=1 << 16):
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        raw = np.empty(cols, np.float32)
        sm = np.empty(cols, np.float32)
        ft = np.empty(2, np.float32)
        act = np.empty(cols, np.int32)
        na = np.zeros(1, np.int32)
        boxes = np.empty(4 * cap, np.float64)
        bins = np.empty(4 * cap, np.int32)
        n = self._chk(self.L.ref_detect(tf.reshape(-1), rows, cols, start_seq, fs, window, order,
                                        margin_db, min_area, int(along_time), raw, sm, ft, act, na,
                                        boxes, bins, cap))
        return dict(raw=raw, smoothed=sm, noise_floor=float(ft[0]), threshold=float(ft[1]),
                    active=act[: na[0]].copy(), boxes=boxes[: 4 * n].reshape(n, 4).copy(),
                    bin_boxes=bins[: 4 * n].reshape(n, 4).copy())

    # ---- signals
    def synthesize(self, scenario_json: str):
        js = scenario_json.encode()
        ns = self._chk(self.L.ref_scenario_samples(js))
        iq = np.empty(ns, np.complex64)
        truth = np.empty(5 * 4096, np.float64)
        nt = _ll(0)
        n = self._chk(self.L.ref_synthesize(js, iq.ctypes.data_as(C.c_void_p), ns, truth, 4096,
                                            C.byref(nt)))
        return iq[:n], truth[: 5 * nt.value].reshape(nt.value, 5).copy()

    def iou(self, a, b) -> float:
        return float(self.L.ref_iou(np.asarray(a, np.float64), np.asarray(b, np.float64)))

    # ---- CPU baseline
    def bench_detect(self, samples, fs, n_fft, rows, n_plots, n_threads):
        iq = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        secs = C.c_double(0.0)
        boxes = self._chk(self.L.ref_bench_detect(iq, len(samples), fs, n_fft, rows, n_plots,
                                                  n_threads, C.byref(secs)))
        return boxes, secs.value

    def run_engine(self, samples, fs, n_fft, rows, n_plots, n_compute, n_sensing):
        iq = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        stats = np.zeros(8, np.float64)
        boxes = self._chk(self.L.ref_run_engine(iq, len(samples), fs, n_fft, rows, n_plots,
                                                n_compute, n_sensing, stats))
        keys = ["plots", "overruns", "wall_s", "p50_s", "p99_s", "fraction_met", "fft_time_s"]
        return boxes, dict(zip(keys, stats.tolist()))

    def summarize(self, plot_index, latency, met, overruns, deadline):
        """runtime::summarize + RunReport::ccdf on scripted records."""
        n = len(latency)
        pi = np.ascontiguousarray(plot_index, np.uint64)
        lat = np.ascontiguousarray(latency, np.float64)
        m = np.ascontiguousarray(met, np.int32)
        stats = np.zeros(10, np.float64)
        cc = np.zeros(2 * max(n, 1), np.float64)
        k = self._chk(self.L.ref_summarize(n, pi.ctypes.data_as(C.POINTER(C.c_ulonglong)), lat, m, overruns,
                                           deadline, stats, cc, max(n, 1)))
        keys = ["plots", "overruns", "deadline_s", "fraction_met", "realtime_met", "p50_s", "p90_s", "p99_s",
                "max_s", "percentiles_valid"]
        return dict(zip(keys, stats.tolist())), [tuple(x) for x in cc[: 2 * k].reshape(-1, 2).tolist()]

    def kernel_sizes(self, rows, cols, conv=2.0, rate=0.5, offset=3.0, mkr=0, mkc=0):
        out = np.zeros(2 * 4096, np.int32)
        n = self._chk(self.L.ref_kernel_sizes(rows, cols, conv, rate, offset, mkr, mkc, out, 4096))
        return out[: 2 * n].reshape(-1, 2)

    def baseline_detect(self, tf, start_seq=0, fs=1e6, conv=2.0, rate=0.5, offset=3.0, mkr=0, mkc=0, cap=1 << 16):
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        boxes = np.zeros(4 * cap, np.float64)
        n = self._chk(self.L.ref_baseline_detect(tf.reshape(-1), rows, cols, start_seq, fs, conv, rate, offset, mkr,
                                                 mkc, boxes, cap))
        return boxes[: 4 * n].reshape(-1, 4)

    def run_engine_boxes(self, samples, fs, n_fft, rows, n_plots, n_compute=2, n_sensing=4, cap=1 << 16):
        """The reference engine (runtime::run, unpaced MemorySource) -> {plot_index: boxes (n,4)}."""
        iq = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        plots = np.zeros(cap, np.uint64)
        boxes = np.zeros(4 * cap, np.float64)
        seen = C.c_ulonglong(0)
        n = self._chk(self.L.ref_run_engine_boxes(iq, len(samples), fs, n_fft, rows, n_plots, n_compute, n_sensing,
                                                  plots.ctypes.data_as(C.POINTER(C.c_ulonglong)), boxes, cap,
                                                  C.byref(seen)))
        out = {}
        b = boxes[: 4 * n].reshape(-1, 4)
        for i in range(n):
            out.setdefault(int(plots[i]), []).append(b[i])
        return {k: np.array(v) for k, v in out.items()}, int(seen.value)


class _Ora:
    def __init__(self):
        L = _load(ORA_SO)
        self.L = L
        sig = {
            "oracle_tf_plot": ([C.c_void_p, C.c_int, C.c_int, C.c_int, _f32p], C.c_int),
            "oracle_psd": ([_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p], C.c_int),
            "oracle_stft_plot": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f32p], C.c_int),
            "oracle_savgol_weights": ([C.c_int, C.c_int, _f64p], C.c_int),
            "oracle_savgol_smooth": ([_f32p, C.c_int, C.c_int, C.c_int, _f32p], C.c_int),
            "oracle_floor_prune": ([_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f32p, _f32p,
                                    _f32p, _i32p], C.c_int),
            "oracle_otsu": ([_f32p, C.c_int, _f32p], C.c_int),
            "oracle_binarize_columns": ([_f32p, C.c_int, C.c_int, _i32p, C.c_int, C.c_int, C.c_int,
                                         _u8p], C.c_int),
            "oracle_morphology": ([_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p], C.c_int),
            "oracle_consolidate": ([_u8p, C.c_int, C.c_int, C.c_int, _u8p], C.c_int),
            "oracle_components": ([_u8p, C.c_int, C.c_int, C.c_int, C.c_void_p, _i64p, _ll], _ll),
            "oracle_detect": ([_f32p, C.c_int, C.c_int, C.c_ulonglong, C.c_double, C.c_int,
                               C.c_int, C.c_double, C.c_int, C.c_int, _f32p, _f32p, _f32p, _i32p,
                               _i32p, _f64p, _i32p, _ll], _ll),
            "oracle_log10f_batch": ([_f32p, _ll, C.c_int, _f32p], None),
            "oracle_powf10_batch": ([_f32p, _ll, C.c_int, _f32p], None),
            "oracle_glibc_log10f_batch": ([_f32p, _ll, _f32p], None),
            "oracle_glibc_powf10_batch": ([_f32p, _ll, _f32p], None),
            "oracle_ssfft_table": ([C.c_int, _f64p], None),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res

    @staticmethod
    def _chk(rc):
        if rc < 0:
            raise OracleError(rc, "restatement rejected the input")
        return rc

    def tf_plot(self, iq: np.ndarray, n_fft: int, rows: int) -> np.ndarray:
        """iq: complex64 (f32 IQ) or int16 array of shape (2*N,) interleaved."""
        iq = np.ascontiguousarray(iq)
        fmt = 1 if iq.dtype == np.int16 else 0
        if fmt == 0:
            iq = iq.astype(np.complex64, copy=False)
        out = np.empty((rows, n_fft), np.float32)
        self._chk(self.L.oracle_tf_plot(iq.ctypes.data_as(C.c_void_p), fmt, n_fft, rows,
                                        out.reshape(-1)))
        return out

    def stft_plot(self, iq: np.ndarray, n_fft: int, hop: int, window: int, rows: int) -> np.ndarray:
        iq = np.ascontiguousarray(iq)
        fmt = 1 if iq.dtype == np.int16 else 0
        if fmt == 0:
            iq = iq.astype(np.complex64, copy=False)
        out = np.empty((rows, n_fft), np.float32)
        self._chk(self.L.oracle_stft_plot(iq.ctypes.data_as(C.c_void_p), fmt, n_fft, hop, window, rows,
                                          out.reshape(-1)))
        return out

    def psd(self, tf, c0=0, c1=None):
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        c1 = cols if c1 is None else c1
        out = np.empty(max(c1 - c0, 1), np.float32)
        self._chk(self.L.oracle_psd(tf.reshape(-1), rows, cols, c0, c1, out))
        return out[: c1 - c0]

    def savgol_weights(self, window, order):
        w = np.empty(window, np.float64)
        self._chk(self.L.oracle_savgol_weights(window, order, w))
        return w

    def savgol_smooth(self, v, window, order):
        v = np.ascontiguousarray(v, np.float32)
        out = np.empty(len(v), np.float32)
        self._chk(self.L.oracle_savgol_smooth(v, len(v), window, order, out))
        return out

    def floor_prune(self, raw, window=31, order=3, margin_db=3.0):
        raw = np.ascontiguousarray(raw, np.float32)
        sm = np.empty(len(raw), np.float32)
        f = np.empty(1, np.float32)
        t = np.empty(1, np.float32)
        act = np.empty(len(raw), np.int32)
        n = self._chk(self.L.oracle_floor_prune(raw, len(raw), window, order, margin_db, sm, f, t,
                                                act))
        return sm, float(f[0]), float(t[0]), act[:n].copy()

    def otsu(self, v):
        v = np.ascontiguousarray(v, np.float32)
        thr = np.zeros(1, np.float32)
        valid = self._chk(self.L.oracle_otsu(v, len(v), thr))
        return bool(valid), float(thr[0])

    def binarize_columns(self, tf, active, c0=0, c1=None, mask=None):
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        c1 = cols if c1 is None else c1
        act = np.ascontiguousarray(active, np.int32)
        m = np.zeros((rows, cols), np.uint8) if mask is None else np.ascontiguousarray(mask, np.uint8)
        self._chk(self.L.oracle_binarize_columns(tf.reshape(-1), rows, cols, act, len(act), c0, c1,
                                                 m.reshape(-1)))
        return m

    def morphology(self, src, op, se):
        src = np.ascontiguousarray(src, np.uint8)
        d = np.zeros_like(src)
        self._chk(self.L.oracle_morphology(src.reshape(-1), src.shape[0], src.shape[1], op, se[0],
                                           se[1], d.reshape(-1)))
        return d

    def consolidate(self, src, along_time=False):
        src = np.ascontiguousarray(src, np.uint8)
        d = np.zeros_like(src)
        self._chk(self.L.oracle_consolidate(src.reshape(-1), src.shape[0], src.shape[1],
                                            int(along_time), d.reshape(-1)))
        return d

    def components(self, mask, min_area, with_labels=True):
        mask = np.ascontiguousarray(mask, np.uint8)
        rows, cols = mask.shape
        cap = min(rows * cols // 2 + 2, 1 << 20)
        ext = np.zeros(5 * cap, np.int64)
        labels = np.zeros((rows, cols), np.int32) if with_labels else None
        n = self._chk(self.L.oracle_components(
            mask.reshape(-1), rows, cols, min_area,
            labels.ctypes.data_as(C.c_void_p) if with_labels else None, ext, cap))
        return ext[: 5 * n].reshape(n, 5), labels

    def detect(self, tf, start_seq=0, fs=1e6, window=31, order=3, margin_db=3.0, min_area=4,
               along_time=False, cap=1 << 16):
        tf = np.ascontiguousarray(tf, np.float32)
        rows, cols = tf.shape
        raw = np.empty(cols, np.float32)
        sm = np.empty(cols, np.float32)
        ft = np.empty(2, np.float32)
        act = np.empty(cols, np.int32)
        na = np.zeros(1, np.int32)
        boxes = np.empty(4 * cap, np.float64)
        bins = np.empty(4 * cap, np.int32)
        n = self._chk(self.L.oracle_detect(tf.reshape(-1), rows, cols, start_seq, fs, window, order,
                                           margin_db, min_area, int(along_time), raw, sm, ft, act,
                                           na, boxes, bins, cap))
        return dict(raw=raw, smoothed=sm, noise_floor=float(ft[0]), threshold=float(ft[1]),
                    active=act[: na[0]].copy(), boxes=boxes[: 4 * n].reshape(n, 4).copy(),
                    bin_boxes=bins[: 4 * n].reshape(n, 4).copy())

    def log10f(self, x, fma=1):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.L.oracle_log10f_batch(x, len(x), fma, out)
        return out

    def powf10(self, y, fma=1):
        y = np.ascontiguousarray(y, np.float32)
        out = np.empty_like(y)
        self.L.oracle_powf10_batch(y, len(y), fma, out)
        return out

    def glibc_log10f(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.L.oracle_glibc_log10f_batch(x, len(x), out)
        return out

    def glibc_powf10(self, y):
        y = np.ascontiguousarray(y, np.float32)
        out = np.empty_like(y)
        self.L.oracle_glibc_powf10_batch(y, len(y), out)
        return out

    def ssfft_table(self, n):
        out = np.empty(2 * n, np.float64)
        self.L.oracle_ssfft_table(n, out)
        return out.reshape(n, 2)


_ref = None
_ora = None


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ora() -> _Ora:
    global _ora
    if _ora is None:
        _ora = _Ora()
    return _ora
