"""paper_2407_07308_b200 -- B200-native BoostCom hot path (BGV word-wise comparison).

Thin Python binding over the C ABI of ``libboostcom.so`` (include/boostcom.h): argument
marshalling only.  Every arithmetic step runs in the library's sm_100a kernels; PyTorch
provides device memory (ciphertexts, workspaces) and streams.  There is no CPU fallback:
importing this package fails if the extension is missing, and every call raises if the
library reports an error.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("BC_LIB_PATH") or os.path.join(_HERE, "libboostcom.so")

if not os.path.exists(_SO):
    raise ImportError("libboostcom.so not built: run __graft_entry__.build() "
                      "(python paper_2407_07308_b200/_build.py)")

_lib = ctypes.CDLL(_SO)


_SCHEDULES = {"r16": 16, "r23": 23, "r26": 26, "r27": 27}    # digit-circuit readings (R16 / R23 / R26 / R27)


class bc_params(ctypes.Structure):
    _fields_ = [("p", ctypes.c_uint32), ("m", ctypes.c_uint32), ("circuit", ctypes.c_char),
                ("d", ctypes.c_uint32), ("l", ctypes.c_uint32),
                ("n_cipher", ctypes.c_uint32), ("cipher_bits", ctypes.c_uint32),
                ("n_special", ctypes.c_uint32), ("special_bits", ctypes.c_uint32),
                ("alpha", ctypes.c_uint32), ("compact_span", ctypes.c_uint32), ("schedule", ctypes.c_uint32),
                ("bluestein", ctypes.c_uint32)]


class bc_info(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in
                ("n", "m", "M", "D", "S", "ints_per_ct", "n_cipher", "n_special", "dnum", "g",
                 "base", "n_galois")]


class bc_ct(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("batch", ctypes.c_uint32), ("level", ctypes.c_uint32)]


class bc_handle(ctypes.Structure):
    _fields_ = [("event", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("consumed", ctypes.c_int)]


_vp, _u32, _u64, _sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
_st = ctypes.c_int


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("bc_ctx_create", _st, ctypes.POINTER(bc_params), ctypes.c_int, ctypes.POINTER(_vp))
_sig("bc_ctx_destroy", None, _vp)
_sig("bc_ctx_info", _st, _vp, ctypes.POINTER(bc_info))
_sig("bc_ctx_moduli", _st, _vp, _vp, _vp)
_sig("bc_ctx_slots", _st, _vp, _vp, _vp, _vp)
_sig("bc_ctx_galois", _st, _vp, _vp)
_sig("bc_ct_bytes", _sz, _vp, _u32, _u32)
_sig("bc_workspace_bytes", _sz, _vp, _u32)
_sig("bc_keygen", _st, _vp, _u64, ctypes.POINTER(_vp), ctypes.POINTER(_vp))
_sig("bc_sk_destroy", None, _vp)
_sig("bc_keys_destroy", None, _vp)
_sig("bc_encrypt", _st, _vp, _vp, _vp, _u32, _u64, _u64, bc_ct, _vp, _sz, _vp)
_sig("bc_encrypt_slots", _st, _vp, _vp, _vp, _u32, _u64, _u64, bc_ct, _vp, _sz, _vp)
_sig("bc_decrypt_slots", _st, _vp, _vp, bc_ct, _vp, _vp, _sz, _vp)
_sig("bc_decrypt", _st, _vp, _vp, bc_ct, _vp, ctypes.c_int, _vp, _sz, _vp)
_sig("bc_decrypt_poly", _st, _vp, _vp, bc_ct, _vp, _vp, _sz, _vp)
_sig("bc_compare", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_compare_lt", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_compare_eq", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_select", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_min", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_max", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_compare_out_level", _u32, _vp, _u32, ctypes.c_int)
_sig("bc_host_stage_bytes", _sz, _vp, _u32, _u32)
_sig("bc_compare_lt_host", _st, _vp, _vp, _vp, _vp, _u32, _u32, _vp, _u32, _vp, _sz, _vp, _sz, _vp)
_sig("bc_compare_lt_async", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp, ctypes.POINTER(bc_handle))
_sig("bc_wait", _st, ctypes.POINTER(bc_handle), _vp)
_sig("bc_ntt_fwd", _st, _vp, _vp, _vp, _u32, _u32, _u32, _vp, _sz, _vp)
_sig("bc_ntt_inv", _st, _vp, _vp, _vp, _u32, _u32, _u32, _vp, _sz, _vp)
_sig("bc_tensor", _st, _vp, bc_ct, bc_ct, _vp, _vp)
_sig("bc_automorph", _st, _vp, bc_ct, _u32, bc_ct, _vp)
_sig("bc_keyswitch", _st, _vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _sz, _vp)
_sig("bc_modswitch", _st, _vp, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_mul", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, _vp, _sz, _vp)
_sig("bc_rotate", _st, _vp, _vp, bc_ct, ctypes.c_int32, bc_ct, _vp, _sz, _vp)
_sig("bc_frobenius", _st, _vp, _vp, bc_ct, _u32, bc_ct, _vp, _sz, _vp)
_sig("bc_extract", _st, _vp, _vp, bc_ct, _vp, _vp, _sz, _vp)
_sig("bc_launch_count", _u64, ctypes.c_int)
_sig("bc_circuit_plan", _st, _u32, ctypes.c_char, _u32, ctypes.POINTER(_u32), ctypes.POINTER(_u32), ctypes.POINTER(_u32))
_sig("bc_ntt_timing", ctypes.c_int, _vp, _vp, _vp)
_sig("bc_phase_timing", ctypes.c_int, _vp, _vp)
_sig("bc_ntt_timing_split", ctypes.c_int, _vp, _vp, _vp, _vp)
_sig("bc_set_ntt_impl", None, ctypes.c_int)
_sig("bc_tune", ctypes.c_int, ctypes.c_char_p, ctypes.c_int64)
_sig("bc_last_error", ctypes.c_char_p)
_sig("bc_min_tree", _st, _vp, _vp, _vp, _u32, bc_ct, _vp, _sz, _vp)
_sig("bc_max_tree", _st, _vp, _vp, _vp, _u32, bc_ct, _vp, _sz, _vp)
_sig("bc_sort", _st, _vp, _vp, _vp, _u32, _vp, _vp, _sz, _vp)
_sig("bc_vec_out_level", _u32, _vp, ctypes.c_int, _vp, _u32)
_sig("bc_vec_workspace_bytes", _sz, _vp, ctypes.c_int, _vp, _u32, _u32)
_sig("bc_private_query_level", _u32, _vp, _u32, _u32, _u32, _u32, _u32)
_sig("bc_private_query_workspace_bytes", _sz, _vp, _u32, _u32, _u32, _u32, _u32, ctypes.c_int)
_sig("bc_private_query", _st, _vp, _vp, bc_ct, bc_ct, bc_ct, bc_ct, _u32, bc_ct, _vp, _sz, _vp, _sz, _vp, _vp)
_sig("bc_graph_capture_begin", _st, _vp)
_sig("bc_graph_capture_end", _st, _vp, ctypes.POINTER(_vp))
_sig("bc_graph_launch", _st, _vp, _vp)
_sig("bc_graph_destroy", None, _vp)
_sig("bc_compact_plan", _st, _u32, _u32, _u32, _vp, _u32, _vp, ctypes.POINTER(_u32))
_sig("bc_compact", _st, _vp, _vp, bc_ct, _vp, bc_ct, ctypes.POINTER(_u32), _vp, _vp, _sz, _vp)

EXPORTS = [n for n in dir(_lib) if n.startswith("bc_")]
if os.environ.get("BC_NTT_GROUP_MB"):
    _lib.bc_tune(b"ntt_group_bytes", int(os.environ["BC_NTT_GROUP_MB"]) << 20)
if os.environ.get("BC_NTT_IMPL"):
    _lib.bc_set_ntt_impl(int(os.environ["BC_NTT_IMPL"]))
for _kv in filter(None, os.environ.get("BC_TUNE", "").split(",")):   # "key=value,..." -> bc_tune (A/B runs)
    _k, _, _v = _kv.partition("=")
    if _lib.bc_tune(_k.strip().encode(), int(_v)) != 0:
        raise ValueError("BC_TUNE: unknown knob " + _k)


class BoostComError(RuntimeError):
    pass


def _check(status, what):
    if status != 0:
        msg = _lib.bc_last_error()
        raise BoostComError("%s failed (status %d): %s" % (what, status, msg.decode() if msg else ""))


def set_ntt_impl(impl):
    """0 = register-blocked NTT passes (default), 1 = radix-2 reference passes."""
    _lib.bc_set_ntt_impl(int(impl))


def ntt_timing(enable=None, split=False):
    """enable/disable live NTT event timing; with enable=None collect -> (ms, limb_transforms, calls)
    (split=True: (ms, limb_transforms, inverse_limb_transforms, calls))."""
    if split and enable is None:
        ms, j, ji, c = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        if _lib.bc_ntt_timing_split(ctypes.byref(ms), ctypes.byref(j), ctypes.byref(ji), ctypes.byref(c)) != 0:
            raise BoostComError("bc_ntt_timing_split failed")
        return ms.value, j.value, ji.value, c.value
    if enable is not None:
        _lib.bc_tune(b"ntt_timing", 1 if enable else 0)
        return None
    ms, j, c = ctypes.c_double(0), ctypes.c_uint64(0), ctypes.c_uint64(0)
    if _lib.bc_ntt_timing(ctypes.byref(ms), ctypes.byref(j), ctypes.byref(c)) != 0:
        raise BoostComError("bc_ntt_timing failed")
    return ms.value, j.value, c.value


PHASES = ("extract", "digit_circuit", "lexicographic", "broadcast_select", "compaction", "private_query_main")


def phase_timing(enable=None):
    """enable/disable per-phase event timing; with enable=None collect -> {phase: (ms, calls)}"""
    if enable is not None:
        _lib.bc_tune(b"phase_timing", 1 if enable else 0)
        return None
    ms = (ctypes.c_double * 6)()
    calls = (ctypes.c_uint64 * 6)()
    if _lib.bc_phase_timing(ms, calls) != 0:
        raise BoostComError("bc_phase_timing failed")
    return {k: (ms[i], int(calls[i])) for i, k in enumerate(PHASES)}


def circuit_plan(p, circuit, schedule="r16"):
    """host only: (k, products per digit, depth) of the digit circuit (R16: k = 0; R23: the selected
    baby-step size)"""
    k, mu, de = _u32(), _u32(), _u32()
    _check(_lib.bc_circuit_plan(int(p), circuit.encode(), _SCHEDULES[schedule], ctypes.byref(k), ctypes.byref(mu),
                                ctypes.byref(de)), "bc_circuit_plan")
    return k.value, mu.value, de.value


class Graph:
    """A CUDA graph of library calls (bc_graph_*): `with Graph() as g: ctx.compare_lt(...)` records the
    calls issued on the current torch stream (which must not be the default stream); g.launch() replays
    them on the same buffers."""

    def __init__(self):
        self._g = None
        self._st = None

    def __enter__(self):
        self._st = _stream()
        _check(_lib.bc_graph_capture_begin(self._st), "bc_graph_capture_begin")
        return self

    def __exit__(self, et, ev, tb):
        g = _vp()
        st = _lib.bc_graph_capture_end(self._st, ctypes.byref(g))
        if et is None:
            _check(st, "bc_graph_capture_end")
            self._g = g
        return False

    def launch(self, stream=None):
        _check(_lib.bc_graph_launch(self._g, stream if stream is not None else _stream()), "bc_graph_launch")

    def __del__(self):
        if self._g is not None and _lib is not None:
            _lib.bc_graph_destroy(self._g)
            self._g = None


def compact_plan(useful, span=3, wpr=None):
    """host only: the library's R17 plan of a usefulness matrix [nin][ints] -> (dest [nin][ints], n_out)"""
    useful = np.ascontiguousarray(useful, dtype=np.uint8)
    nin, ints = useful.shape
    dest = np.zeros((nin, ints), dtype=np.int32)
    n = _u32()
    _check(_lib.bc_compact_plan(ints, span, wpr or ints, useful.ctypes.data, nin, dest.ctypes.data, ctypes.byref(n)),
           "bc_compact_plan")
    return dest, n.value


def launch_count(reset=False):
    return int(_lib.bc_launch_count(1 if reset else 0))


def _torch():
    import torch
    return torch


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class Keys:
    def __init__(self, ctx, sk, keys):
        self.ctx, self.sk, self.keys = ctx, sk, keys

    def __del__(self):
        try:
            _lib.bc_sk_destroy(self.sk)
            _lib.bc_keys_destroy(self.keys)
        except Exception:
            pass


class Context:
    """One parameter set on one CUDA device (R1-R17 of DESIGN.md)."""

    def __init__(self, cfg, device=0):
        torch = _torch()
        self.device = torch.device("cuda", device)
        prm = bc_params(int(cfg["p"]), int(cfg["m"]), cfg.get("circuit", "U").encode(), int(cfg["d"]),
                        int(cfg["l"]), int(cfg["n_cipher"]), int(cfg["cipher_bits"]),
                        int(cfg["n_special"]), int(cfg["special_bits"]), int(cfg["alpha"]),
                        int(cfg.get("compact_span", 3)), _SCHEDULES[cfg.get("schedule", "r16")],
                        {"pow2": 0, "mixed": 1}[cfg.get("bluestein", "pow2")])
        h = _vp()
        with torch.cuda.device(self.device):
            _check(_lib.bc_ctx_create(ctypes.byref(prm), device, ctypes.byref(h)), "bc_ctx_create")
        self._h = h
        info = bc_info()
        _check(_lib.bc_ctx_info(h, ctypes.byref(info)), "bc_ctx_info")
        self.info = {k: getattr(info, k) for k, _ in bc_info._fields_}
        for k, v in self.info.items():
            setattr(self, k, v)
        self.cfg = dict(cfg)
        self.p = int(cfg["p"])
        self.d, self.l = int(cfg["d"]), int(cfg["l"])
        self._ws = None

    def __del__(self):
        try:
            _lib.bc_ctx_destroy(self._h)
        except Exception:
            pass

    # ---- tables ----
    def moduli(self):
        k = self.n_cipher + self.n_special
        a = np.zeros(k, dtype=np.uint64)
        w = np.zeros(k, dtype=np.uint64)
        _check(_lib.bc_ctx_moduli(self._h, a.ctypes.data, w.ctypes.data), "bc_ctx_moduli")
        return [int(x) for x in a], [int(x) for x in w]

    def slots(self):
        G = np.zeros(self.D + 1, dtype=np.int64)
        z = np.zeros(self.D, dtype=np.int64)
        t = np.zeros(self.S, dtype=np.int64)
        _check(_lib.bc_ctx_slots(self._h, G.ctypes.data, z.ctypes.data, t.ctypes.data), "bc_ctx_slots")
        return G, z, t

    def galois(self):
        g = np.zeros(self.n_galois, dtype=np.uint32)
        _check(_lib.bc_ctx_galois(self._h, g.ctypes.data), "bc_ctx_galois")
        return [int(x) for x in g]

    # ---- memory ----
    def ct_empty(self, batch, level, parts=2):
        torch = _torch()
        return torch.empty((batch, parts, level, self.n), dtype=torch.int64, device=self.device)

    def workspace(self, nbytes):
        torch = _torch()
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = None
            self._ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        return self._ws

    def default_ws(self, batch=1):
        need = _lib.bc_workspace_bytes(self._h, batch)
        return self.workspace(max(need, 1 << 26))

    def _wsargs(self, ws):
        if ws is None:
            ws = self._ws if self._ws is not None else self.default_ws(1)
        return _ptr(ws), ws.numel()

    @staticmethod
    def view(t):
        assert t.dtype.itemsize == 8 and t.is_contiguous() and t.dim() == 4 and t.shape[1] == 2
        return bc_ct(t.data_ptr(), t.shape[0], t.shape[2])

    def workspace_bytes(self, batch):
        return int(_lib.bc_workspace_bytes(self._h, batch))

    def out_level(self, level, which=0):
        return int(_lib.bc_compare_out_level(self._h, level, which))

    # ---- keys / encryption ----
    def keygen(self, seed):
        sk, k = _vp(), _vp()
        _check(_lib.bc_keygen(self._h, seed, ctypes.byref(sk), ctypes.byref(k)), "bc_keygen")
        return Keys(self, sk, k)

    def encrypt(self, keys, words, seed, ct_index0=0, ws=None):
        words = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1, self.ints_per_ct)
        B = words.shape[0]
        out = self.ct_empty(B, self.n_cipher)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_encrypt(self._h, keys.keys, words.ctypes.data, B, seed, ct_index0, self.view(out), w, wb,
                               _stream()), "bc_encrypt")
        return out

    def encrypt_slots(self, keys, slots, seed, ct_index0=0, ws=None):
        slots = np.ascontiguousarray(slots, dtype=np.int16).reshape(-1, self.S, self.D)
        B = slots.shape[0]
        out = self.ct_empty(B, self.n_cipher)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_encrypt_slots(self._h, keys.keys, slots.ctypes.data, B, seed, ct_index0, self.view(out), w,
                                     wb, _stream()), "bc_encrypt_slots")
        return out

    def decrypt(self, keys, ct, as_bits=False, ws=None):
        B = ct.shape[0]
        out = np.zeros((B, self.ints_per_ct), dtype=np.uint64)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_decrypt(self._h, keys.sk, self.view(ct), out.ctypes.data, 1 if as_bits else 0, w, wb,
                               _stream()), "bc_decrypt")
        return out

    def decrypt_slots(self, keys, ct, ws=None):
        B = ct.shape[0]
        out = np.zeros((B, self.S, self.D), dtype=np.int16)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_decrypt_slots(self._h, keys.sk, self.view(ct), out.ctypes.data, w, wb, _stream()),
               "bc_decrypt_slots")
        return out

    def decrypt_poly(self, keys, ct, ws=None):
        B = ct.shape[0]
        out = np.zeros((B, self.n), dtype=np.int64)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_decrypt_poly(self._h, keys.sk, self.view(ct), out.ctypes.data, w, wb, _stream()),
               "bc_decrypt_poly")
        return out

    # ---- comparison ----
    def _cmp(self, fn, keys, a, b, which, ws):
        lvl = self.out_level(min(a.shape[2], b.shape[2]), which)
        out = self.ct_empty(a.shape[0], lvl)
        w, wb = self._wsargs(ws)
        _check(fn(self._h, keys.keys, self.view(a), self.view(b), self.view(out), w, wb, _stream()), fn.__name__)
        return out

    def compare_lt(self, keys, a, b, ws=None):
        return self._cmp(_lib.bc_compare_lt, keys, a, b, 0, ws)

    def compare_lt_host(self, keys, h_a, h_b, h_out, chunk=0, ws=None, stage=None):
        """bc_compare_lt_host: compare_lt of host (pinned) ciphertext tensors into the host tensor h_out,
        host<->device copies pipelined with the compare on a library copy stream (end-to-end path)."""
        B, lvl = h_a.shape[0], h_a.shape[2]
        ch = chunk or max(1, (B + 3) // 4)
        need = int(_lib.bc_host_stage_bytes(self._h, ch, lvl))
        if stage is None:                # its own buffer: the compare workspace must not alias it
            stage = _torch().empty(need, dtype=_torch().uint8, device=self.device)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_compare_lt_host(self._h, keys.keys, h_a.data_ptr(), h_b.data_ptr(), B, lvl, h_out.data_ptr(), ch,
                                       stage.data_ptr(), stage.numel() * stage.element_size(), w, wb, _stream()),
               "bc_compare_lt_host")
        return h_out

    def compare_eq(self, keys, a, b, ws=None):
        return self._cmp(_lib.bc_compare_eq, keys, a, b, 1, ws)

    def min(self, keys, a, b, ws=None):
        return self._cmp(_lib.bc_min, keys, a, b, 2, ws)

    def max(self, keys, a, b, ws=None):
        return self._cmp(_lib.bc_max, keys, a, b, 2, ws)

    def compare(self, keys, a, b, ws=None):
        lvl = min(a.shape[2], b.shape[2])
        lt = self.ct_empty(a.shape[0], self.out_level(lvl, 0))
        eq = self.ct_empty(a.shape[0], self.out_level(lvl, 1))
        w, wb = self._wsargs(ws)
        _check(_lib.bc_compare(self._h, keys.keys, self.view(a), self.view(b), self.view(lt), self.view(eq), w, wb,
                               _stream()), "bc_compare")
        return lt, eq

    def private_query(self, keys, data, q, codes, op1, e, side_stream=None, ws=None, ws_side=None, out=None):
        """R24 private_q (Listings 3-5): blocking when side_stream is None, else the branch
        evaluation runs on side_stream (non-blocking).  Returns the result batch (current stream)."""
        lvl = int(_lib.bc_private_query_level(self._h, data.shape[0], data.shape[2], q.shape[2], op1.shape[2], e))
        if lvl == 0:
            raise BoostComError("bc_private_query_level failed")
        if out is None:
            out = self.ct_empty(data.shape[0], lvl)
        if ws is None:
            ws = self.workspace(int(_lib.bc_private_query_workspace_bytes(self._h, data.shape[0], data.shape[2],
                                                                          q.shape[2], op1.shape[2], e, 0)))
        sp, sb, ss = None, 0, None
        if side_stream is not None:
            if ws_side is None:
                torch = _torch()
                ws_side = torch.empty(int(_lib.bc_private_query_workspace_bytes(
                    self._h, data.shape[0], data.shape[2], q.shape[2], op1.shape[2], e, 1)), dtype=torch.uint8,
                    device=self.device)
            sp, sb, ss = _ptr(ws_side), ws_side.numel(), ctypes.c_void_p(side_stream.cuda_stream)
        _check(_lib.bc_private_query(self._h, keys.keys, self.view(data), self.view(q), self.view(codes),
                                     self.view(op1), int(e), self.view(out), _ptr(ws), ws.numel(), sp, sb, _stream(),
                                     ss), "bc_private_query")
        return out

    def compare_lt_async(self, keys, a, b, out, side_stream, ws):
        h = bc_handle()
        _check(_lib.bc_compare_lt_async(self._h, keys.keys, self.view(a), self.view(b), self.view(out), _ptr(ws),
                                        ws.numel(), ctypes.c_void_p(side_stream.cuda_stream), ctypes.byref(h)),
               "bc_compare_lt_async")
        return h

    @staticmethod
    def wait(h, joiner_stream):
        return _lib.bc_wait(ctypes.byref(h), ctypes.c_void_p(joiner_stream.cuda_stream))

    def select(self, keys, cond, x1, x2, ws=None):
        torch = _torch()
        # output level: mul(bcast(cond), diff) -> min level - 1
        lvl = min(cond.shape[2], x1.shape[2], x2.shape[2]) - 1
        out = self.ct_empty(x1.shape[0], lvl)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_select(self._h, keys.keys, self.view(cond), self.view(x1), self.view(x2), self.view(out), w,
                              wb, _stream()), "bc_select")
        del torch
        return out

    # ---- vectors: tournament / sort (R20, R21) ----
    _VEC = {"min": 0, "max": 1, "sort": 2}

    def vec_out_level(self, op, levels):
        lv = np.ascontiguousarray(levels, dtype=np.uint32)
        r = int(_lib.bc_vec_out_level(self._h, self._VEC[op], lv.ctypes.data, len(lv)))
        if r == 0:
            raise BoostComError("bc_vec_out_level: no valid schedule for %s over levels %s" % (op, list(levels)))
        return r

    def vec_workspace_bytes(self, op, levels, batch):
        lv = np.ascontiguousarray(levels, dtype=np.uint32)
        return int(_lib.bc_vec_workspace_bytes(self._h, self._VEC[op], lv.ctypes.data, len(lv), batch))

    def _vec(self, op, keys, elems, ws):
        T = len(elems)
        views = (bc_ct * T)(*[self.view(e) for e in elems])
        levels = [e.shape[2] for e in elems]
        lvl = self.vec_out_level(op, levels)
        nout = T if op == "sort" else 1
        outs = [self.ct_empty(elems[0].shape[0], lvl) for _ in range(nout)]
        if ws is None:
            ws = self.workspace(self.vec_workspace_bytes(op, levels, elems[0].shape[0]))
        w, wb = _ptr(ws), ws.numel()
        ov = (bc_ct * nout)(*[self.view(o) for o in outs])
        if op == "sort":
            _check(_lib.bc_sort(self._h, keys.keys, views, T, ov, w, wb, _stream()), "bc_sort")
            return outs
        fn = _lib.bc_min_tree if op == "min" else _lib.bc_max_tree
        _check(fn(self._h, keys.keys, views, T, ov[0], w, wb, _stream()), fn.__name__)
        return outs[0]

    def min_tree(self, keys, elems, ws=None):
        """R20 slot-wise min over the T ciphertext batches `elems` (fixed tree)."""
        return self._vec("min", keys, elems, ws)

    def max_tree(self, keys, elems, ws=None):
        return self._vec("max", keys, elems, ws)

    def sort(self, keys, elems, ws=None):
        """R21 slot-wise rank sort of T <= p ciphertext batches -> T outputs (ascending)."""
        return self._vec("sort", keys, elems, ws)

    # ---- primitives (parity tests) ----
    def ntt_fwd(self, x, prime0=0, ws=None):
        """x: int64 tensor [npoly, nlimb, n] (coefficient residues) -> evaluation form."""
        out = x.new_empty(x.shape)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_ntt_fwd(self._h, _ptr(x), _ptr(out), x.shape[0], x.shape[1], prime0, w, wb, _stream()),
               "bc_ntt_fwd")
        return out

    def ntt_inv(self, x, prime0=0, ws=None):
        out = x.new_empty(x.shape)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_ntt_inv(self._h, _ptr(x), _ptr(out), x.shape[0], x.shape[1], prime0, w, wb, _stream()),
               "bc_ntt_inv")
        return out

    def tensor(self, a, b):
        torch = _torch()
        out = torch.empty((a.shape[0], 3, a.shape[2], self.n), dtype=torch.int64, device=self.device)
        _check(_lib.bc_tensor(self._h, self.view(a), self.view(b), _ptr(out), _stream()), "bc_tensor")
        return out

    def automorph(self, a, t):
        out = a.new_empty(a.shape)
        _check(_lib.bc_automorph(self._h, self.view(a), t, self.view(out), _stream()), "bc_automorph")
        return out

    def keyswitch(self, keys, d, t, ws=None):
        """d: [B, level, n] evaluation form -> (u0, u1) as [B, 2, level, n]."""
        torch = _torch()
        B, lvl = d.shape[0], d.shape[1]
        out = torch.empty((B, 2, lvl, self.n), dtype=torch.int64, device=self.device)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_keyswitch(self._h, keys.keys, _ptr(d), B, lvl, t, _ptr(out), w, wb, _stream()),
               "bc_keyswitch")
        return out

    def modswitch(self, a, ws=None):
        out = self.ct_empty(a.shape[0], a.shape[2] - 1)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_modswitch(self._h, self.view(a), self.view(out), w, wb, _stream()), "bc_modswitch")
        return out

    def mul(self, keys, a, b, ws=None):
        out = self.ct_empty(a.shape[0], min(a.shape[2], b.shape[2]) - 1)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_mul(self._h, keys.keys, self.view(a), self.view(b), self.view(out), w, wb, _stream()),
               "bc_mul")
        return out

    def rotate(self, keys, a, k, ws=None):
        out = a.new_empty(a.shape)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_rotate(self._h, keys.keys, self.view(a), k, self.view(out), w, wb, _stream()), "bc_rotate")
        return out

    def frobenius(self, keys, a, k, ws=None):
        out = a.new_empty(a.shape)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_frobenius(self._h, keys.keys, self.view(a), k, self.view(out), w, wb, _stream()),
               "bc_frobenius")
        return out

    def extract(self, keys, a, ws=None):
        torch = _torch()
        out = torch.empty((a.shape[0], self.d, 2, a.shape[2], self.n), dtype=torch.int64, device=self.device)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_extract(self._h, keys.keys, self.view(a), _ptr(out), w, wb, _stream()), "bc_extract")
        return out

    def compact(self, keys, cts, useful, ws=None):
        """-> (compacted cts at level-1, dest[n_in, ints] destination block or -1)."""
        useful = np.ascontiguousarray(useful, dtype=np.uint8).reshape(cts.shape[0], self.ints_per_ct)
        out = self.ct_empty(cts.shape[0], cts.shape[2] - 1)
        nout = _u32(0)
        dest = np.zeros(useful.shape, dtype=np.int32)
        w, wb = self._wsargs(ws)
        _check(_lib.bc_compact(self._h, keys.keys, self.view(cts), useful.ctypes.data, self.view(out),
                               ctypes.byref(nout), dest.ctypes.data, w, wb, _stream()), "bc_compact")
        return out[: nout.value], dest


def load_params(name_or_path):
    """params/<name>.json (or a path); "<name>@pow2" / "@mixed" sets the Bluestein length (R25),
    "<name>@r16" / "@r23" the digit circuits (R16 / R23)"""
    import json
    name, _, opt = name_or_path.partition("@")
    path = name
    if not os.path.exists(path):
        path = os.path.join(_HERE, "..", "params", name + ".json")
    with open(path) as f:
        cfg = json.load(f)
    if opt in ("pow2", "mixed"):
        cfg["bluestein"] = opt
    elif opt:
        cfg["schedule"] = opt
    return cfg


# ------------------------------------------------------------------------------------------
# roofline probe of the dominant kernel family (Bluestein NTT passes)
# ------------------------------------------------------------------------------------------
SMS = 148
FP64_PER_SM_PER_CLK = 64          # B200 DFMA lanes per SM per clock: measured 18.2e12/s (tools/micro/bfly_micro.cu)
FP64_PER_MODBFLY = 8              # one modular butterfly in binary64 (ntt3.cu): DMUL + 3 DFMA + 2 DADD (product) + 2 DADD
IMAD_PER_SM_PER_CLK = 64          # integer path (ntt2.cu, impl 7): IMAD issue rate per SM (guide)
IMAD_PER_MULMOD = 10              # 64-bit Shoup product: mul.hi.u64 (4) + 2 x mul.lo.u64 (3): SASS-checked


def ntt_peak(sm_mhz=1965.0):
    """peak modular butterflies (or pointwise products) per second of the binary64 NTT, in T/s"""
    return SMS * FP64_PER_SM_PER_CLK * sm_mhz * 1e6 / FP64_PER_MODBFLY / 1e12


def ntt_work(ctx):
    """algorithmic 64-bit modular multiplications of one limb-transform (forward Bluestein):
    two size-M NTTs (M/2 log2 M butterflies each; log2 of a mixed-radix length M = 256 r N' taken as is),
    the pointwise D^ product (M), two chirps (n+m)."""
    import math
    M = ctx.M
    return int(round(M * math.log2(M))) + M + ctx.n + ctx.m


def barrett_work(ctx):
    """extra algorithmic work of an inverse limb-transform at composite m: the Barrett division by Phi_m
     runs one size-Mb cyclic convolution (Mb log2 Mb butterflies + Mb pointwise products),
    Mb = the smallest power of two >= max(2(m - n) - 1, m); the sparse quotient (a few shifted adds) is
    not counted.  0 for prime m."""
    import math
    m, n = ctx.m, ctx.n
    if m - n == 1:
        return 0
    Mb = 1
    while Mb < max(2 * (m - n) - 1, m):
        Mb *= 2
    return Mb * int(math.log2(Mb)) + Mb


def profile_ntt(ctx, npoly=64, reps=5, sm_mhz=1965.0):
    torch = _torch()
    L = ctx.n_cipher
    g = torch.Generator(device=ctx.device)
    g.manual_seed(1)
    x = torch.randint(0, 1 << 40, (npoly, L, ctx.n), dtype=torch.int64, device=ctx.device, generator=g)
    out = torch.empty_like(x)
    scratch = ctx.workspace(max(npoly * L * ctx.M * 8 + (1 << 22), 1 << 26))
    st = _stream()
    for _ in range(2):
        _check(_lib.bc_ntt_fwd(ctx._h, _ptr(x), _ptr(out), npoly, L, 0, _ptr(scratch), scratch.numel(), st), "ntt")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _check(_lib.bc_ntt_fwd(ctx._h, _ptr(x), _ptr(out), npoly, L, 0, _ptr(scratch), scratch.numel(), st), "ntt")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    work = npoly * L * ntt_work(ctx)
    achieved = work / (ms / 1e3) / 1e12
    peak = ntt_peak(sm_mhz)
    traffic = None
    try:
        import json
        prof = os.path.join(_HERE, "..", "profiles", "r1_ntt_probe_ncu.json")
        if npoly == 64 and ctx.n == 30940 and os.path.exists(prof):
            traffic = json.load(open(prof))["traffic_bytes_per_probe_launch"]
    except Exception:
        traffic = None
    return {"bound": "alu", "kernel": "bluestein_ntt (passA+passB+passC)", "achieved": achieved, "peak": peak,
            "unit": "T modmul/s", "frac": achieved / peak, "traffic": traffic,
            "traffic_note": "DRAM bytes per probe launch from profiles/r1_ntt_probe_ncu.json (ncu --set full)",
            "per_launch_ms": ms, "limb_transforms_per_launch": npoly * L,
            "work_per_limb_transform": ntt_work(ctx),
            "peak_note": "148 SM x 64 DFMA/clk x %.0f MHz / %d FP64 ops per modular butterfly" % (sm_mhz, FP64_PER_MODBFLY)}
