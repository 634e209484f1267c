"""B200 (sm_100a) hot path of Checkmate two-phase rounding (arXiv:1910.02653).

Thin Python binding over the C ABI of include/cm.h -- argument marshalling only;
every step of the path (rounding, R closure, FREE, U peak, cost, per-budget
argmin) runs in libcheckmate_b200.so.  PyTorch supplies device memory and
streams.  Importing fails loudly when the shared library is missing.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._abi import (CM_EMAX, CM_KEY_NONE, CM_LAYOUT_BLK, CM_LAYOUT_DENSE, CM_LAYOUT_TRI4,  # noqa: F401
                   CM_ROUND_RANDOMIZED,
                   CM_ROUND_THRESHOLD,
                   CM_NMAX)

_lib = _abi.load()


class CMError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.cm_status_string(status).decode()
        detail = _lib.cm_last_error().decode()
        super().__init__(f"{where}: {msg}" + (f" ({detail})" if detail else ""))


def _check(status: int, where: str):
    if status != _abi.CM_OK:
        raise CMError(status, where)


LAYOUTS = {"dense": CM_LAYOUT_DENSE, "tri4": CM_LAYOUT_TRI4, "blk": CM_LAYOUT_BLK}


def sstar_floats(n: int, layout: str, ld: int = 0) -> int:
    """cm_sstar_floats: floats one S* occupies in a layout (the minimum stride)."""
    return int(_lib.cm_sstar_floats(int(n), LAYOUTS[layout], int(ld)))


def tri4_size(n: int) -> int:
    return sstar_floats(n, "tri4")


class Graph:
    """Device-resident DAG (cm_graph).  pred_ptr/pred_idx: CSR of DEPS(k), 0-based."""

    def __init__(self, n, pred_ptr, pred_idx, cost, mem, ovh):
        self.n = int(n)
        pp = np.ascontiguousarray(pred_ptr, np.int32)
        pi = np.ascontiguousarray(pred_idx, np.int32)
        c = np.ascontiguousarray(cost, np.int64)
        m = np.ascontiguousarray(mem, np.int64)
        h = ctypes.c_void_p()
        st = _lib.cm_graph_create(self.n, pp.ctypes.data, pi.ctypes.data if pi.size else None,
                                  c.ctypes.data, m.ctypes.data, int(ovh), ctypes.byref(h))
        _check(st, "cm_graph_create")
        self._h = h
        self.pred_ptr, self.pred_idx, self.cost, self.mem, self.ovh = pp, pi, c, m, int(ovh)
        self.cost_bound = int(_lib.cm_graph_cost_bound(h))

    @classmethod
    def from_edges(cls, n, edges, cost, mem, ovh):
        ptr = np.zeros(n + 1, np.int32)
        for (_, j) in edges:
            ptr[j + 1] += 1
        ptr = np.cumsum(ptr).astype(np.int32)
        idx = np.zeros(len(edges), np.int32)
        fill = ptr[:-1].copy()
        for (i, j) in sorted(edges, key=lambda e: (e[1], e[0])):
            idx[fill[j]] = i
            fill[j] += 1
        return cls(n, ptr, idx, cost, mem, ovh)

    @classmethod
    def from_workload(cls, g):
        return cls.from_edges(g.n, g.edges, g.cost, g.mem, g.ovh)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            _lib.cm_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def key_idx_bits(total_candidates: int) -> int:
    return int(_lib.cm_key_idx_bits(int(total_candidates)))


def decode_key(key: int, idx_bits: int):
    c = ctypes.c_int64()
    i = ctypes.c_int64()
    _lib.cm_decode_key(int(key), int(idx_bits), ctypes.byref(c), ctypes.byref(i))
    return int(c.value), int(i.value)


def decode_batch_key(key: int, idx_bits: int):
    """max-batch key -> (B_max, idx); (0, -1) when nothing fits (cm_decode_batch_key)."""
    b = ctypes.c_int64()
    i = ctypes.c_int64()
    _lib.cm_decode_batch_key(int(key), int(idx_bits), ctypes.byref(b), ctypes.byref(i))
    return b.value, i.value


POLICIES = {"all": 0, "sqrt": 1, "greedy": 2, "ap_sqrt": 3, "ap_greedy": 4}


def policy_checkpoints(graph: Graph, L: int, policy: str, b: int = 0) -> np.ndarray:
    """cm_policy_checkpoints: the checkpoint set (uint8 [L]) of a baseline policy (Table 1)."""
    out = np.zeros(int(L), np.uint8)
    st = _lib.cm_policy_checkpoints(graph.n, int(L), graph.pred_ptr.ctypes.data,
                                    graph.pred_idx.ctypes.data if graph.pred_idx.size else None,
                                    graph.mem.ctypes.data, POLICIES[policy], int(b), out.ctypes.data)
    if st != _abi.CM_OK:
        raise CMError(st, "cm_policy_checkpoints: " + _lib.cm_policy_last_error().decode())
    return out


def baseline_sweep(graph: Graph, L: int, specs, budget=None, ld: int | None = None, stream=None):
    """Evaluate baseline policies in one batch: specs = [(policy, b)];
    the checkpoint sets are built on the host, their S matrices written on the device
    (cm_policy_sstar) and evaluated like rounded S* (theta = 0.5).  Returns round_and_evaluate's
    dict plus "k_sets" (uint8 [len(specs)][L])."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    ld = int(ld) if ld else -(-graph.n // 32) * 32
    k = np.stack([policy_checkpoints(graph, L, p, b) for (p, b) in specs])
    kd = torch.from_numpy(k).to(dev)
    sstar = torch.empty((len(specs), graph.n, ld), dtype=torch.float32, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    _check(_lib.cm_policy_sstar(graph.handle, int(L), len(specs), kd.data_ptr(), sstar.data_ptr(), ld,
                                ctypes.c_void_p(stream)), "cm_policy_sstar")
    out = round_and_evaluate(graph, sstar, torch.tensor([0.5], dtype=torch.float32, device=dev), budget,
                             stream=stream)
    out["k_sets"] = k
    out["sstar"] = sstar
    return out


CM_OP_COMPUTE, CM_OP_DEALLOC = 0, 1


def emit_plan(n, pred_ptr, pred_idx, mem, mem_overhead, r_rows, s_rows, hoist: bool = True):
    """cm_emit_plan: Alg. 1 execution plan, optionally hoisted,
    for one candidate's R / S masks (host uint64 [n][W], the layout round_and_evaluate returns).
    Returns (statements, peak): statements as (op, stage, node, reg) tuples, 0-based."""
    pred_ptr = np.ascontiguousarray(pred_ptr, np.int32)
    pred_idx = np.ascontiguousarray(pred_idx, np.int32)
    mem = np.ascontiguousarray(mem, np.int64)
    r = np.ascontiguousarray(r_rows).view(np.uint64)
    s = np.ascontiguousarray(s_rows).view(np.uint64)
    cap = int(2 * r.size * 64 + 16)
    while True:
        out = np.zeros((cap, 4), np.int32)
        cnt, peak = ctypes.c_int64(), ctypes.c_int64()
        st = _lib.cm_emit_plan(int(n), pred_ptr.ctypes.data, pred_idx.ctypes.data if pred_idx.size else None,
                               mem.ctypes.data, int(mem_overhead), r.ctypes.data, s.ctypes.data, int(bool(hoist)),
                               out.ctypes.data, cap, ctypes.byref(cnt), ctypes.byref(peak))
        if st == _abi.CM_ERANGE and cnt.value > cap:
            cap = cnt.value
            continue
        if st != _abi.CM_OK:
            raise CMError(st, "cm_emit_plan: " + _lib.cm_plan_last_error().decode())
        return [tuple(int(v) for v in row) for row in out[:cnt.value]], int(peak.value)


def debug_trace(max_values: int = 4096):
    """(k1_begin, k1_end, k2_begin, k2_end) per chunk of the last CM_TRACE=1 call, in ms."""
    buf = (ctypes.c_float * max_values)()
    m = _lib.cm_debug_trace(buf, max_values)
    return [tuple(buf[i:i + 4]) for i in range(0, m, 4)]



def debug_cta_trace(back: int = 0, max_values: int = 4 * 1024):
    """CM_TRACE=2 per-CTA %globaltimer stamps of the calling thread's fused call `back` calls ago:
    uint64 [CTAs][4] = {start, rounding warps done, ~(first unit-0 wait satisfied), scan warps done}."""
    buf = (ctypes.c_uint64 * max_values)()
    m = _lib.cm_debug_cta_trace_at(int(back), buf, max_values)
    return np.frombuffer(buf, np.uint64, count=m).reshape(-1, 4).copy()


def last_call_seq(graph: Graph) -> int:
    """cm_last_call_seq: the number of the graph's last round_and_evaluate call."""
    return int(_lib.cm_last_call_seq(graph.handle))


def stream_wait_call(graph: Graph, seq: int, stream) -> None:
    """cm_stream_wait_call: `stream` (a CUDA stream handle) waits until call `seq` on `graph`
    has written all its outputs (a stream memory operation; nothing is enqueued on the stream
    the call itself ran on)."""
    _check(_lib.cm_stream_wait_call(graph.handle, int(seq) & 0xffffffff, ctypes.c_void_p(stream)),
           "cm_stream_wait_call")


def debug_last_launches() -> int:
    """Kernels launched by this thread's last round_and_evaluate call (cm_debug_last_launches)."""
    return int(_lib.cm_debug_last_launches())

def _ptr(t):
    return None if t is None else t.data_ptr()


def round_and_evaluate(graph: Graph, sstar, theta, budget=None, *, layout: str = "dense",
                       n_sstar: int | None = None, ld: int | None = None, stride: int | None = None,
                       index_base: int = 0, total_candidates: int | None = None,
                       best_key=None, masks: bool = False, peak=None, cost=None, stream=None,
                       samples: int | None = None, seed: int = 0, cost_limit: int | None = None,
                       best_batch_key=None, init_keys: bool = False, overlap: bool = False,
                       best_key_mc: int | None = None, best_batch_key_mc: int | None = None):
    """cm_round_and_evaluate on device tensors.

    sstar : float32 CUDA tensor; dense [N_S, n, ld], tri4 [N_S, tri4_size(n)] or blk
            [N_S, sstar_floats(n, "blk")] (or any buffer with explicit n_sstar / ld / stride).
    theta : float32 CUDA tensor [N_theta] (deterministic rounding, Alg. 2 line 1), or None with
            ``samples`` = N samples per S* of randomized rounding (R1,
            Philox key ``seed``).
    budget: int64 CUDA tensor [N_B] or None.
    cost_limit: with budgets, also run the max-batch epilogue (Eq. 13; the key of the largest
            B_max per budget among candidates with cost <= cost_limit, in ``best_batch_key``).
    init_keys: the call sets best_key / best_batch_key to CM_KEY_NONE itself (CM_EVAL_INIT_KEYS).
    overlap: the call may start while the previous kernel on the stream drains
            (CM_EVAL_OVERLAP): only when that work writes none of this call's inputs and touches
            none of its outputs, e.g. consecutive calls alternating two output sets.
    best_key_mc / best_batch_key_mc: device addresses (ints) of the NVLink multicast views of
            best_key / best_batch_key (dist.MulticastKeys): the a8 MIN over ranks then happens in
            the reduce step (multimem.red.min); the caller initialises all replicas first.
    Returns dict(peak, cost, best_key, idx_bits, r_mask, s_mask) of CUDA tensors.
    Asynchronous on ``stream`` (default: torch's current stream).
    """
    import torch
    n = graph.n
    lay = LAYOUTS[layout]
    if n_sstar is None:
        n_sstar = sstar.shape[0]
    if lay == CM_LAYOUT_DENSE:
        if ld is None:
            ld = sstar.shape[-1]
        if stride is None:
            stride = n * ld if sstar.dim() < 3 else sstar.stride(0)
    else:
        ld = 0
        if stride is None:
            stride = sstar.stride(0) if sstar.dim() == 2 else sstar_floats(n, layout)
    dev = sstar.device
    randomized = samples is not None
    if randomized == (theta is not None):
        raise ValueError("give exactly one of theta (deterministic) and samples (randomized)")
    n_theta = int(samples) if randomized else theta.numel()
    n_cand = n_sstar * n_theta
    n_budget = 0 if budget is None else budget.numel()
    if overlap and (peak is None or cost is None or (n_budget and best_key is None)
                    or (cost_limit is not None and n_budget and best_batch_key is None)):
        # an overlapped call may still be running the previous call's tail: outputs allocated
        # here could reuse memory the caller just dropped that the previous call still writes
        raise ValueError("overlap=True needs caller-owned peak, cost and best_key (and best_batch_key) "
                         "that no call still in flight writes")
    if total_candidates is None:
        total_candidates = index_base + n_cand
    if peak is None:
        peak = torch.empty(n_cand, dtype=torch.int64, device=dev)
    if cost is None:
        cost = torch.empty(n_cand, dtype=torch.int64, device=dev)
    if best_key is None and n_budget:
        best_key = torch.full((n_budget,), CM_KEY_NONE, dtype=torch.int64, device=dev)
    if cost_limit is not None and best_batch_key is None and n_budget:
        best_batch_key = torch.full((n_budget,), CM_KEY_NONE, dtype=torch.int64, device=dev)
    r_mask = s_mask = None
    if masks:
        W = (n + 63) // 64
        r_mask = torch.zeros((n_cand, n, W), dtype=torch.int64, device=dev)
        s_mask = torch.zeros((n_cand, n, W), dtype=torch.int64, device=dev)
    a = _abi.EvalArgs()
    a.n_sstar = n_sstar
    a.layout = lay
    a.sstar = sstar.data_ptr()
    a.ld = int(ld)
    a.sstar_stride = int(stride)
    a.n_theta = n_theta
    a.theta = None if randomized else theta.data_ptr()
    a.rounding = _abi.CM_ROUND_RANDOMIZED if randomized else _abi.CM_ROUND_THRESHOLD
    a.seed = int(seed) & ((1 << 64) - 1)
    a.best_batch_key = _ptr(best_batch_key)
    a.cost_limit = int(cost_limit) if cost_limit is not None else 0
    a.flags = (_abi.CM_EVAL_INIT_KEYS if init_keys else 0) | (_abi.CM_EVAL_OVERLAP if overlap else 0)
    a.n_budget = n_budget
    a.budget = _ptr(budget)
    a.index_base = int(index_base)
    a.total_candidates = int(total_candidates)
    a.peak = peak.data_ptr()
    a.cost = cost.data_ptr()
    a.best_key = _ptr(best_key)
    a.r_mask = _ptr(r_mask)
    a.s_mask = _ptr(s_mask)
    a.best_key_mc = int(best_key_mc) if best_key_mc else None
    a.best_batch_key_mc = int(best_batch_key_mc) if best_batch_key_mc else None
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    _check(_lib.cm_round_and_evaluate(graph.handle, ctypes.byref(a), ctypes.c_void_p(stream)),
           "cm_round_and_evaluate")
    return {"peak": peak, "cost": cost, "best_key": best_key, "best_batch_key": best_batch_key,
            "idx_bits": key_idx_bits(total_candidates), "r_mask": r_mask, "s_mask": s_mask}


class HostPipeline:
    """End-to-end path for S* batches in (pinned) HOST memory.

    The batch is cut into chunks; chunk c is copied host->device on a copy stream into
    one of two device buffers while the kernel evaluates chunk c-1 on the compute stream
    (double buffering with CUDA events), then peak / cost / keys come back device->host.
    Device buffers are allocated once here, not per call."""

    def __init__(self, graph: Graph, row_floats: int, chunk: int, n_theta: int, n_budget: int,
                 layout: str = "tri4", ld: int | None = None, device="cuda"):
        import torch
        self.graph, self.chunk, self.layout = graph, int(chunk), layout
        self.ld, self.row_floats = ld, int(row_floats)
        self.dev = torch.device(device)
        self.bufs = [torch.empty((self.chunk, self.row_floats), dtype=torch.float32, device=self.dev)
                     for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(self.dev)
        self.compute_stream = torch.cuda.Stream(self.dev)
        self.n_theta, self.n_budget = n_theta, n_budget

    def run(self, host_sstar, theta, budget=None, index_base: int = 0, total_candidates=None):
        """host_sstar: pinned CPU float32 tensor [N_S, row_floats]; theta / budget: CUDA tensors.
        Returns (peak, cost, best_key) as CPU tensors (synchronised)."""
        import torch
        N = host_sstar.shape[0]
        n_cand = N * self.n_theta
        total = index_base + n_cand if total_candidates is None else total_candidates
        peak = torch.empty(n_cand, dtype=torch.int64, device=self.dev)
        cost = torch.empty(n_cand, dtype=torch.int64, device=self.dev)
        key = None
        if budget is not None:
            key = torch.full((budget.numel(),), CM_KEY_NONE, dtype=torch.int64, device=self.dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        cs, ks = self.copy_stream, self.compute_stream
        ks.wait_stream(torch.cuda.current_stream(self.dev))
        for c, s0 in enumerate(range(0, N, self.chunk)):
            cnt = min(self.chunk, N - s0)
            b = c & 1
            buf = self.bufs[b]
            with torch.cuda.stream(cs):
                if c >= 2:
                    cs.wait_event(freed[b])
                buf[:cnt].copy_(host_sstar[s0:s0 + cnt], non_blocking=True)
                copied[b].record(cs)
            with torch.cuda.stream(ks):
                ks.wait_event(copied[b])
                lo, hi = s0 * self.n_theta, (s0 + cnt) * self.n_theta
                round_and_evaluate(self.graph, buf, theta, budget, layout=self.layout, n_sstar=cnt,
                                   ld=self.ld, stride=self.row_floats, index_base=index_base + lo,
                                   total_candidates=total, best_key=key, peak=peak[lo:hi],
                                   cost=cost[lo:hi], stream=ks.cuda_stream)
                freed[b].record(ks)
        with torch.cuda.stream(ks):
            out = (peak.to("cpu", non_blocking=True), cost.to("cpu", non_blocking=True),
                   None if key is None else key.to("cpu", non_blocking=True))
        ks.synchronize()
        return out
