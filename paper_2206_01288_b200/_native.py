"""ctypes binding of lib/libhetsched_sm100a.so (the C-ABI in include/hetsched_b200.h).

There is no fallback: if the library or a CUDA device is missing, every
entry point raises NativeUnavailable.  Device buffers are handed over as raw
pointers of torch CUDA tensors; torch is plumbing only.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from collections import OrderedDict
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libhetsched_sm100a.so"
# experiments only: load an alternative build of the same sources
if os.environ.get("HS_LIB_PATH"):
    LIB_PATH = Path(os.environ["HS_LIB_PATH"]).resolve()
SOURCES = sorted((PKG / "csrc").glob("*.cu")) + sorted((PKG / "csrc").glob("*.cuh")) + sorted(
    (PKG / "csrc").glob("*.h")) + [PKG.parent / "include" / "hetsched_b200.h"]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is not available."""


class NativeError(RuntimeError):
    """A C-ABI call returned an error code."""


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu under csrc/ (in parallel, one object each) and link
    lib/libhetsched_sm100a.so for sm_100a."""
    newest = max(p.stat().st_mtime for p in SOURCES)
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= newest:
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor
    objdir = LIB_PATH.parent / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + os.environ.get("HS_NVCC_EXTRA", "").split()
    cus = sorted((PKG / "csrc").glob("*.cu"))

    def deps(cu: Path) -> set:
        """cu plus the local headers it includes, transitively."""
        seen, todo = set(), [cu]
        while todo:
            f = todo.pop()
            if f in seen or not f.exists():
                continue
            seen.add(f)
            for ln in f.read_text().splitlines():
                ln = ln.strip()
                if ln.startswith('#include "'):
                    name = ln.split('"')[1]
                    for base in (f.parent, PKG.parent / "include"):
                        if (base / name).exists():
                            todo.append(base / name)
                            break
        return seen

    def one(cu: Path):
        obj = objdir / (cu.stem + ".o")
        if not force and obj.exists() and obj.stat().st_mtime >= max(d.stat().st_mtime for d in deps(cu)):
            return obj, subprocess.CompletedProcess([], 0, "", "")
        r = subprocess.run([nvcc, *compile_flags, "-c", "-o", str(obj), str(cu)], capture_output=not verbose,
                           text=True)
        return obj, r

    with ThreadPoolExecutor(max_workers=max(1, min(len(cus), os.cpu_count() or 1))) as ex:
        results = list(ex.map(one, cus))
    errs = [r.stderr for _, r in results if r.returncode]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    tmp = LIB_PATH.with_suffix(".so.tmp")
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
                        *[str(o) for o, _ in results]], capture_output=not verbose, text=True)
    if r.returncode:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class PCG64(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_int32), ("uinteger", C.c_uint32)]

    @classmethod
    def from_generator(cls, rng: np.random.Generator) -> "PCG64":
        st = rng.bit_generator.state
        if st.get("bit_generator") != "PCG64":
            raise TypeError("the GPU search reproduces numpy's PCG64 stream only")
        s, inc = st["state"]["state"], st["state"]["inc"]
        M = (1 << 64) - 1
        return cls(s >> 64, s & M, inc >> 64, inc & M, st["has_uint32"], st["uinteger"])

    def write_back(self, rng: np.random.Generator) -> None:
        st = rng.bit_generator.state
        st["state"]["state"] = (int(self.state_hi) << 64) | int(self.state_lo)
        st["has_uint32"] = int(self.has_uint32)
        st["uinteger"] = int(self.uinteger)
        rng.bit_generator.state = st


class GAConfig(C.Structure):
    _fields_ = [("pop_size", C.c_int32), ("generations", C.c_int32), ("kind", C.c_int32),
                ("max_passes", C.c_int32), ("patience", C.c_int32)]


_lock = threading.Lock()
_lib = None


def lib():
    """Load the library once; raise NativeUnavailable if it cannot run here."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeUnavailable(f"{LIB_PATH} is missing; run __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.hs_version.restype = i32
        L.hs_last_error.restype = C.c_char_p
        L.hs_instance_create.argtypes = [vp, vp, i32, i32, i32, dbl, dbl, dbl, i32, C.POINTER(vp)]
        L.hs_instance_destroy.argtypes = [vp]
        L.hs_instance_tables.argtypes = [vp, vp, vp, vp]
        L.hs_eval_batch.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]
        L.hs_eval_batch_host.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp]
        L.hs_eval_batch_ex.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp, i32, vp]
        L.hs_path_heuristic_batch.argtypes = [vp, i32, i64, vp, vp, i32, vp]
        L.hs_bottleneck_batch.argtypes = [vp, i32, i64, vp, i32, vp]
        L.hs_path_batch.argtypes = [vp, i32, i64, vp, vp, i32, vp]
        pcg = C.POINTER(PCG64)
        L.hs_ga_create.argtypes = [vp, C.POINTER(GAConfig), i32, pcg, C.POINTER(vp)]
        L.hs_ga_create_ex.argtypes = [vp, C.POINTER(GAConfig), i32, pcg, i32, C.POINTER(vp)]
        L.hs_ga_run.argtypes = [vp, i32, vp]
        L.hs_ga_export.argtypes = [vp, i32, vp, vp, vp]
        L.hs_ga_import.argtypes = [vp, i32, vp, vp, vp, vp]
        L.hs_ga_result.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, pcg]
        L.hs_ga_destroy.argtypes = [vp]
        L.hs_local_search.argtypes = [vp, i32, i32, i32, vp, pcg, vp, vp, vp]
        L.hs_refine_pass.argtypes = [vp, i32, i32, i32, vp, pcg, vp, vp]
        L.hs_crossover.argtypes = [i32, i32, i32, i32, i32, vp, vp, pcg, vp]
        L.hs_gains.argtypes = [i32, i32, i32, i32, vp, i32, i32, vp, vp, vp]
        L.hs_random_partitions.argtypes = [i32, i32, i32, i32, i32, pcg, vp]
        L.hs_materialize.argtypes = [vp, i64, vp, vp, vp]
        L.hs_evaluate_assignments.argtypes = [vp, i64, vp, vp, vp]
        L.hs_random_assignments.argtypes = [i32, i32, i32, i32, i32, pcg, vp, vp]
        L.hs_count_partitions.argtypes = [i32, i32]
        L.hs_bottleneck_match_batch.argtypes = [vp, i32, i64, vp, vp, i32, vp]
        L.hs_datap_group_batch.argtypes = [vp, vp, i32, i64, dbl, dbl, vp, i32, vp]
        L.hs_brute_force.argtypes = [vp, i32, i32, vp, vp, i32, vp]
        L.hs_unrank_partitions.argtypes = [i32, i32, i32, i64, i64, vp, vp]
        L.hs_probe_smem_bandwidth.argtypes = [i32, vp, vp]
        for name in EXPORTS:
            if name not in ("hs_version", "hs_last_error"):
                getattr(L, name).restype = i32
        L.hs_count_partitions.restype = i64
        _lib = L
        return L


EXPORTS = ("hs_version", "hs_last_error", "hs_instance_create", "hs_instance_destroy", "hs_instance_tables",
           "hs_eval_batch", "hs_eval_batch_ex", "hs_eval_batch_host", "hs_path_heuristic_batch",
           "hs_bottleneck_batch", "hs_path_batch", "hs_ga_create", "hs_ga_create_ex", "hs_ga_run",
           "hs_ga_export", "hs_ga_import", "hs_ga_result", "hs_ga_destroy", "hs_local_search", "hs_refine_pass",
           "hs_crossover", "hs_gains", "hs_random_partitions", "hs_materialize", "hs_evaluate_assignments",
           "hs_random_assignments", "hs_count_partitions", "hs_unrank_partitions", "hs_bottleneck_match_batch",
           "hs_datap_group_batch", "hs_brute_force", "hs_probe_smem_bandwidth")


def smem_bandwidth(device: int = 0) -> float:
    """Measured shared-memory bandwidth of the GPU, bytes/s (hs_probe.cu)."""
    out = np.zeros(2)
    check(lib().hs_probe_smem_bandwidth(device, out.ctypes.data, out[1:].ctypes.data), "hs_probe_smem_bandwidth")
    return float(out[0])


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().hs_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def torch_cuda():
    """torch with a visible CUDA device, or NativeUnavailable."""
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise NativeUnavailable("torch is required for device buffers") from exc
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the hetsched GPU path has no CPU fallback")
    return torch


def current_device() -> int:
    return torch_cuda().cuda.current_device()


def ptr(a) -> int | None:
    """Raw pointer of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def stream_ptr(device: int):
    torch = torch_cuda()
    return torch.cuda.current_stream(device).cuda_stream


class Instance:
    """Device-resident pair tables for one (graph, workload) on one GPU."""

    def __init__(self, lat: np.ndarray, bw: np.ndarray, d_pp: int, d_dp: int, c_pp, c_dp, device: int):
        L = lib()
        torch_cuda()
        self.lat = np.ascontiguousarray(lat, dtype=np.float64)
        self.bw = np.ascontiguousarray(bw, dtype=np.float64)
        self.n, self.k, self.m, self.device = self.lat.shape[0], int(d_pp), int(d_dp), int(device)
        # host-formed numerators, with the reference's own scalar arithmetic
        self.dp_num = float(8.0 * c_dp)
        self.pp_num = float(8.0 * c_pp)
        self.sw_num = float(8.0 * (c_pp + c_dp))
        h = C.c_void_p()
        check(L.hs_instance_create(self.lat.ctypes.data, self.bw.ctypes.data, self.n, self.k, self.m,
                                   self.dp_num, self.pp_num, self.sw_num, self.device, C.byref(h)),
              "hs_instance_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        lib = globals().get("_lib")
        if h is not None and lib is not None:
            lib.hs_instance_destroy(h)
            self.handle = None

    def tables(self):
        n = self.n
        dp, pp, sw = (np.empty((n, n)) for _ in range(3))
        check(lib().hs_instance_tables(self.handle, dp.ctypes.data, pp.ctypes.data, sw.ctypes.data),
              "hs_instance_tables")
        return dp, pp, sw


_cache: "OrderedDict[tuple, tuple]" = OrderedDict()
_cache_lock = threading.Lock()
_CACHE_MAX = 32


def instance_for(g, w, device: int | None = None) -> Instance:
    """Cached Instance for a CommGraph-like ``g`` and WorkloadSpec-like ``w``.

    Read-only arrays (CommGraph freezes them) are keyed by identity and kept
    alive by the cache entry; writeable arrays are keyed by content."""
    if device is None:
        device = current_device()
    lat, bw = g.lat, g.bw
    wkey = (int(w.d_pp), int(w.d_dp), repr(w.c_pp), repr(w.c_dp), int(device))
    if isinstance(lat, np.ndarray) and isinstance(bw, np.ndarray) and not lat.flags.writeable \
            and not bw.flags.writeable:
        key = ("id", id(lat), id(bw)) + wkey
    else:
        import hashlib
        la = np.ascontiguousarray(lat, dtype=np.float64)
        ba = np.ascontiguousarray(bw, dtype=np.float64)
        key = ("sha", hashlib.sha1(la.tobytes() + ba.tobytes()).hexdigest()) + wkey
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            _cache.move_to_end(key)
            return hit[0]
    inst = Instance(lat, bw, w.d_pp, w.d_dp, w.c_pp, w.c_dp, device)
    with _cache_lock:
        _cache[key] = (inst, lat, bw)
        while len(_cache) > _CACHE_MAX:
            _cache.popitem(last=False)
    return inst
