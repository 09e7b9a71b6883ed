"""Operator API of the fused GNN layer path -- the Python mirror of the C++ layer in
include/gnncg/ops.hpp, both sitting on the C ABI of include/gnncg_b200.h.

Names, argument meaning and error behaviour follow the reference's data model
(gnncg::Graph / gnncg::Tensor, head-major multi-head layout, LeakyReLU slope 0.2,
TensorError on shape mismatch, GraphError on bad endpoints) and the operator
contracts of its specified executor:

  gat_forward / gat_backward           GAT layer (App. B)
  edgeconv_forward / edgeconv_backward EdgeConv layer
  gmm_forward / gmm_backward           GMMConv layer
  gcn_forward / gcn_backward / spmm    GCN layer, weighted Aggregate
  matmul / matmul_nt / matmul_tn       dense transforms (tensor.cpp:8-60)

All tensors are fp32 CUDA tensors; every FLOP runs in libgnncg_b200.so.  torch
provides device memory and the current stream only.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._lib import TensorError, call
from .graph import DeviceGraph, _ptr, _stream

DEFAULT_SLOPE = 0.2  # tensor.hpp:93 


class KernelProbe:
    """Optional per-call CUDA-event timing on the launching stream (bench.py roofline).
    Disabled by default; enabling it records two events around each fused / GEMM call."""

    def __init__(self):
        self.enabled = False
        self.pending = []  # (name, start, end)
        self.totals: dict[str, list] = {}

    def __call__(self, name):
        probe = self

        class _Scope:
            def __enter__(self):
                if probe.enabled:
                    self.s = torch.cuda.Event(enable_timing=True)
                    self.e = torch.cuda.Event(enable_timing=True)
                    self.s.record()
                return self

            def __exit__(self, *exc):
                if probe.enabled:
                    self.e.record()
                    probe.pending.append((name, self.s, self.e))
                return False

        return _Scope()

    def collect(self):
        """Synchronise and fold pending events into totals[name] = [ms_sum, count]."""
        torch.cuda.synchronize()
        for name, s, e in self.pending:
            t = self.totals.setdefault(name, [0.0, 0])
            t[0] += s.elapsed_time(e)
            t[1] += 1
        self.pending.clear()
        return self.totals

    def reset(self):
        self.pending.clear()
        self.totals.clear()


PROBE = KernelProbe()


def _f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda:
        raise TensorError(f"{name}: expected a float32 CUDA tensor")
    return t.contiguous()


def _f32_rows(t: torch.Tensor, name: str) -> torch.Tensor:
    """fp32 CUDA matrix with unit column stride; a padded row stride (e.g. 16-byte aligned, which
    the TMA tensor-core GEMM needs) is kept as is."""
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda or t.dim() != 2:
        raise TensorError(f"{name}: expected a 2-D float32 CUDA tensor")
    if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        t = t.contiguous()
    return t


def _shape(t: torch.Tensor, shape, name: str):
    if tuple(t.shape) != tuple(shape):
        raise TensorError(f"{name}: shape {tuple(t.shape)} != expected {tuple(shape)}")
    return t


def _out(t: torch.Tensor, shape, name: str) -> torch.Tensor:
    """A caller-provided output buffer: exact shape, contiguous fp32 CUDA (written by pointer)."""
    _shape(t, shape, name)
    if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
        raise TensorError(f"{name}: expected a contiguous float32 CUDA tensor")
    return t


# ---------------------------------------------------------------------------
# Dense transforms (K1 / K5)
# ---------------------------------------------------------------------------
def gemm(A: torch.Tensor, B: torch.Tensor, trans_a=False, trans_b=False, out: torch.Tensor | None = None,
         ws=None) -> torch.Tensor:
    """C = op(A) op(B) in fp32 on the device (deterministic)."""
    A = _f32_rows(A, "gemm A")
    B = _f32_rows(B, "gemm B")
    M, K = (A.shape[1], A.shape[0]) if trans_a else (A.shape[0], A.shape[1])
    Kb, N = (B.shape[1], B.shape[0]) if trans_b else (B.shape[0], B.shape[1])
    if K != Kb:
        raise TensorError("matmul: inner dimension mismatch")  # tensor.cpp:10
    if out is None:
        out = torch.empty(M, N, dtype=torch.float32, device=A.device)
    need = _lib.lib().gnncg_gemm_workspace(int(trans_a), int(trans_b), M, N, K)
    if ws is None:
        buf = torch.empty(max(need, 1), dtype=torch.uint8, device=A.device)
        wp, wn = buf.data_ptr(), buf.numel()
    else:
        wp, wn = ws.get(need)
    with PROBE(f"gemm_{'t' if trans_a else 'n'}{'t' if trans_b else 'n'}"):
        call("gnncg_gemm", int(trans_a), int(trans_b), M, N, K, _ptr(A), A.stride(0), _ptr(B), B.stride(0),
             _ptr(out), out.stride(0), wp, wn, _stream())
    return out


def matmul(a, b, ws=None):
    """C = A B (tensor.cpp:8-24)."""
    return gemm(a, b, ws=ws)


def matmul_nt(a, b, ws=None):
    """C = A B^T (tensor.cpp:26-42)."""
    return gemm(a, b, trans_b=True, ws=ws)


def matmul_tn(a, b, ws=None):
    """C = A^T B (tensor.cpp:44-60)."""
    return gemm(a, b, trans_a=True, ws=ws)


# ---------------------------------------------------------------------------
# GAT
# ---------------------------------------------------------------------------
@dataclass
class GatParams:
    """heads x f per-head width, LeakyReLU slope.  gather = "fp32" (default: the 1e-4 parity
    contract) or "bf16": the fused kernels gather Ht / dOut rows from bf16 copies (half the
    bytes per edge; all arithmetic, logits and outputs stay fp32) -- the north star's
    "bf16 features" option, held to the looser bound BF16_BOUND."""

    heads: int
    f: int
    slope: float = DEFAULT_SLOPE
    gather: str = "fp32"


BF16_BOUND = 2e-2  # max-normalised relative error of the bf16-gather mode (tests/test_gpu_gat.py)


def _check_gather(p: GatParams) -> bool:
    if p.gather == "fp32":
        return False
    if p.gather != "bf16":
        raise ValueError(f"gather must be 'fp32' or 'bf16', not {p.gather!r}")
    if not _lib.lib().gnncg_gat_bf16_supported(p.heads, p.f):
        raise _lib.UnsupportedError(f"bf16 gather unsupported for heads={p.heads} f={p.f}")
    return True


def pack_bf16(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 -> bf16 (round to nearest even) on the device, as raw int16 storage."""
    x = _f32(x, "pack_bf16 input")
    if out is None:
        out = torch.empty(x.shape, dtype=torch.int16, device=x.device)
    call("gnncg_pack_bf16", x.numel(), _ptr(x), _ptr(out), _stream())
    return out


@dataclass
class GatStash:
    """What the forward keeps for the backward: vertex tensors only (O(|V|)).
    Ht / Al / Ar are the reorganized ApplyVertex outputs; m / d the edge-softmax statistics."""

    Ht: torch.Tensor
    Al: torch.Tensor
    Ar: torch.Tensor
    m: torch.Tensor
    d: torch.Tensor
    out: torch.Tensor | None = None  # the layer output (kept anyway as the next layer's input)
    Ht_lp: torch.Tensor | None = None  # bf16 gather copy of Ht (gather="bf16")


@dataclass
class GatGrads:
    dH: torch.Tensor | None
    dW: torch.Tensor
    da_l: torch.Tensor
    da_r: torch.Tensor


def gat_region_forward(g: DeviceGraph, Ht, Al, Ar, p: GatParams, out=None, m=None, d=None, chunk=None, Ht_lp=None):
    """K2 alone: the fused region given the reorganized vertex tensors (gather="bf16": the rows
    come from Ht_lp, packed here when not given)."""
    V, h, f = g.num_vertices, p.heads, p.f
    Ht, Al, Ar = _f32(Ht, "Ht"), _f32(Al, "A_l"), _f32(Ar, "A_r")
    _shape(Ht, (V, h * f), "Ht")
    _shape(Al, (V, h), "A_l")
    _shape(Ar, (V, h), "A_r")
    dev = Ht.device
    out = torch.empty(V, h * f, device=dev) if out is None else out
    m = torch.empty(V, h, device=dev) if m is None else m
    d = torch.empty(V, h, device=dev) if d is None else d
    idx = g.csr_dst
    sched = idx.sched(chunk) if chunk else idx.sched()
    need = _lib.lib().gnncg_gat_workspace(sched.struct(), None, h, f)
    wp, wn = g.ws.get(need)
    if _check_gather(p):
        Ht_lp = pack_bf16(Ht) if Ht_lp is None else Ht_lp
        with PROBE("gat_fwd"):
            call("gnncg_gat_fwd_bf16", idx.struct(), sched.struct(), h, f, p.slope, _ptr(Ht_lp), _ptr(Al), _ptr(Ar),
                 _ptr(out), _ptr(m), _ptr(d), wp, wn, _stream())
        return out, m, d
    with PROBE("gat_fwd"):
        call("gnncg_gat_fwd", idx.struct(), sched.struct(), h, f, p.slope, _ptr(Ht), _ptr(Al), _ptr(Ar), _ptr(out),
             _ptr(m), _ptr(d), wp, wn, _stream())
    return out, m, d


def attn_dots(Ht, a_l, a_r, heads, f, Al=None, Ar=None):
    V = Ht.shape[0]
    Al = torch.empty(V, heads, device=Ht.device) if Al is None else Al
    Ar = torch.empty(V, heads, device=Ht.device) if Ar is None else Ar
    with PROBE("attn_dots"):
        call("gnncg_gat_attn_dots", V, heads, f, _ptr(Ht), _ptr(_f32(a_l, "a_l")), _ptr(_f32(a_r, "a_r")),
             _ptr(Al), _ptr(Ar), _stream())
    return Al, Ar


def gat_transform(H, W, a_l, a_r, heads, f, ws=None, Ht=None, Al=None, Ar=None):
    """K1 with the attention-LP epilogue: Ht = H W, A_l = Ht . a_l, A_r = Ht . a_r in one
    tensor-core GEMM (gnncg_gat_transform).  Ht / Al / Ar may be given (contiguous, e.g. a
    rank's block of the all-gather tables)."""
    M, K = H.shape
    hf = heads * f
    dev = H.device
    Ht = torch.empty(M, hf, device=dev) if Ht is None else _out(Ht, (M, hf), "Ht")
    Al = torch.empty(M, heads, device=dev) if Al is None else _out(Al, (M, heads), "Al")
    Ar = torch.empty(M, heads, device=dev) if Ar is None else _out(Ar, (M, heads), "Ar")
    need = _lib.lib().gnncg_gemm_workspace(0, 0, M, hf, K)
    if ws is None:
        buf = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
        wp, wn = buf.data_ptr(), buf.numel()
    else:
        wp, wn = ws.get(need)
    with PROBE("gat_transform"):
        call("gnncg_gat_transform", M, K, heads, f, _ptr(H), H.stride(0), _ptr(W), _ptr(Ht), _ptr(a_l), _ptr(a_r),
             _ptr(Al), _ptr(Ar), wp, wn, _stream())
    return Ht, Al, Ar


def gat_forward(g: DeviceGraph, H, W, a_l, a_r, p: GatParams, chunk=None):
    """One GAT layer forward, reorganized:
    Ht = H W (K1), A_l = Ht . a_l, A_r = Ht . a_r, then the fused region (K2).
    Returns (out, GatStash)."""
    h, f = p.heads, p.f
    H, W = _f32_rows(H, "H"), _f32(W, "W")
    if H.shape[0] != g.num_vertices:
        raise TensorError("gat_forward: H rows != num_vertices")
    if W.shape != (H.shape[1], h * f):
        raise TensorError(f"gat_forward: W shape {tuple(W.shape)} != ({H.shape[1]}, {h * f})")
    _shape(a_l, (h, f), "a_l")
    _shape(a_r, (h, f), "a_r")
    Ht, Al, Ar = gat_transform(H, W, _f32(a_l, "a_l"), _f32(a_r, "a_r"), h, f, ws=g.ws)
    Ht_lp = pack_bf16(Ht) if _check_gather(p) else None
    out, m, d = gat_region_forward(g, Ht, Al, Ar, p, chunk=chunk, Ht_lp=Ht_lp)
    return out, GatStash(Ht, Al, Ar, m, d, out, Ht_lp)


def fast_supported(p: GatParams) -> bool:
    return bool(_lib.lib().gnncg_gat_fast_supported(p.heads, p.f))


def gat_region_backward(g: DeviceGraph, stash: GatStash, a_l, a_r, dOut, p: GatParams, chunk=None, mode="auto"):
    """Recompute backward of the fused region: returns (dHt, dAl, dAr, da_l, da_r, c).

    mode "deterministic": K3 over csr_dst then K4 over csc_src, fixed-order sums (bitwise
    reproducible).  mode "fast": the spec's lock-free fast mode -- c from the
    row dot <dOut, out>, then one fused pass over csc_src with dA_r accumulated by global
    reductions (no csr_dst gather pass).  "auto" = fast when supported and stash.out is present."""
    V, h, f = g.num_vertices, p.heads, p.f
    dOut = _f32(dOut, "dOut")
    _shape(dOut, (V, h * f), "dOut")
    a_l, a_r = _f32(a_l, "a_l"), _f32(a_r, "a_r")
    lp = _check_gather(p)
    if mode == "auto":
        mode = "fast" if (stash.out is not None and (lp or fast_supported(p))) else "deterministic"
    if lp and mode != "fast":
        raise TensorError("gather='bf16' needs the fast backward (stash.out)")
    dev = dOut.device
    c = torch.empty(V, h, device=dev)
    dAr = torch.empty(V, h, device=dev)
    dAl = torch.empty(V, h, device=dev)
    dHt = torch.empty(V, h * f, device=dev)
    sd = g.csr_dst.sched(chunk) if chunk else g.csr_dst.sched()
    ss = g.csc_src.sched(chunk) if chunk else g.csc_src.sched()
    L = _lib.lib()
    need = max(L.gnncg_gat_workspace(sd.struct(), ss.struct(), h, f), L.gnncg_gat_attn_grad_workspace(V, h, f))
    wp, wn = g.ws.get(need)
    s = _stream()
    if mode == "fast":
        if stash.out is None:
            raise TensorError("gat_region_backward(fast): stash.out is required")
        rec = torch.empty(V, L.gnncg_gat_rec_stride(h), device=dev)
        if lp:
            # c from the rounded dOut rows K4f gathers (written here), the own row from the same
            # rounded Ht the forward aggregated: the softmax-backward identity stays exact
            dOut_lp = torch.empty(dOut.shape, dtype=torch.int16, device=dev)
            Ht_lp = stash.Ht_lp if stash.Ht_lp is not None else pack_bf16(stash.Ht)
            with PROBE("gat_bwd_prep"):
                call("gnncg_gat_bwd_prep_bf16", V, h, f, _ptr(dOut), _ptr(stash.out), _ptr(stash.Ar), _ptr(stash.m),
                     _ptr(stash.d), _ptr(rec), _ptr(dOut_lp), s)
        else:
            with PROBE("gat_bwd_prep"):
                call("gnncg_gat_bwd_prep", V, h, f, _ptr(dOut), _ptr(stash.out), _ptr(stash.Ar), _ptr(stash.m),
                     _ptr(stash.d), _ptr(rec), s)
        c = rec.view(V, h, 4)[:, :, 2]  # record = float4 {A_r, lse, c, 0} per head
        if lp:
            with PROBE("gat_bwd_src_fused"):
                call("gnncg_gat_bwd_src_fused_bf16", g.csc_src.struct(), ss.struct(), h, f, p.slope, 0, V,
                     _ptr(Ht_lp), _ptr(stash.Al), _ptr(rec), _ptr(dOut_lp), _ptr(a_l), _ptr(a_r), _ptr(dHt),
                     _ptr(dAl), _ptr(dAr), wp, wn, s)
        else:
            with PROBE("gat_bwd_src_fused"):
                call("gnncg_gat_bwd_src_fused", g.csc_src.struct(), ss.struct(), h, f, p.slope, 0, V,
                     _ptr(stash.Ht), _ptr(stash.Al), _ptr(rec), _ptr(dOut), _ptr(a_l), _ptr(a_r), _ptr(dHt),
                     _ptr(dAl), _ptr(dAr), wp, wn, s)
    elif mode == "deterministic":
        with PROBE("gat_bwd_dst"):
            call("gnncg_gat_bwd_dst", g.csr_dst.struct(), sd.struct(), h, f, p.slope, _ptr(stash.Ht),
                 _ptr(stash.Al), _ptr(stash.Ar), _ptr(stash.m), _ptr(stash.d), _ptr(dOut), _ptr(c), _ptr(dAr),
                 wp, wn, s)
        with PROBE("gat_bwd_src"):
            call("gnncg_gat_bwd_src", g.csc_src.struct(), ss.struct(), h, f, p.slope, 0, V, _ptr(stash.Ht),
                 _ptr(stash.Al), _ptr(stash.Ar), _ptr(stash.m), _ptr(stash.d), _ptr(c), _ptr(dOut), _ptr(dAr),
                 _ptr(a_l), _ptr(a_r), _ptr(dHt), _ptr(dAl), wp, wn, s)
    else:
        raise ValueError(f"unknown backward mode {mode!r}")
    da_l = torch.empty(h, f, device=dev)
    da_r = torch.empty(h, f, device=dev)
    with PROBE("attn_grad"):
        call("gnncg_gat_attn_grad", V, h, f, _ptr(stash.Ht), _ptr(dAl), _ptr(dAr), _ptr(da_l), _ptr(da_r), wp, wn,
             s)
    return dHt, dAl, dAr, da_l, da_r, c


def gat_backward(g: DeviceGraph, H, W, a_l, a_r, stash: GatStash, dOut, p: GatParams, need_dH=True, chunk=None,
                 mode="auto"):
    """GAT layer backward with recomputation:
    region backward (K3+K4, or the fused fast pass) -> LP grads -> dW = H^T dHt (K5),
    dH = dHt W^T (K5)."""
    H, W = _f32_rows(H, "H"), _f32(W, "W")
    dHt, _, _, da_l, da_r, _ = gat_region_backward(g, stash, a_l, a_r, dOut, p, chunk=chunk, mode=mode)
    dW = gemm(H, dHt, trans_a=True, ws=g.ws)
    dH = gemm(dHt, W, trans_b=True, ws=g.ws) if need_dH else None
    return GatGrads(dH, dW, da_l, da_r)


# ---------------------------------------------------------------------------
# EdgeConv
# ---------------------------------------------------------------------------
NO_EDGE = 0xFFFFFFFF


@dataclass
class EdgeConvStash:
    Y: torch.Tensor  # [Th | Ph], V x 2C
    argmax: torch.Tensor  # int32 holding u32 edge ids (0xFFFFFFFF = empty row)


def edgeconv_region_forward(g: DeviceGraph, Th, Ph):
    """K6 alone: out, argmax (int32 view of u32 edge ids)."""
    V, C_ = Th.shape
    out = torch.empty(V, C_, device=Th.device)
    amax = torch.empty(V, C_, dtype=torch.int32, device=Th.device)
    with PROBE("edgeconv_fwd"):
        call("gnncg_edgeconv_fwd", g.csr_dst.struct(), C_, 0, _ptr(Th), Th.stride(0), _ptr(Ph), Ph.stride(0), _ptr(out),
             _ptr(amax), _stream())
    return out, amax


def _adjacent_columns(parts, name):
    """When the column blocks `parts` are consecutive slices of one row-major buffer (the
    models keep [Theta | Phi] and [W | P_l | P_r] that way), that buffer as one matrix view --
    no copy; else None."""
    A = parts[0]
    if not all(isinstance(p, torch.Tensor) and p.is_cuda and p.dtype == torch.float32 and p.dim() == 2 for p in parts):
        raise TensorError(f"{name}: expected 2-D float32 CUDA tensors")
    ld = A.stride(0)
    col = 0
    for p in parts:
        if p.stride(1) != 1 or p.stride(0) != ld or p.shape[0] != A.shape[0] or p.data_ptr() != A.data_ptr() + 4 * col:
            return None
        col += p.shape[1]
    if col > ld:
        return None
    return A.as_strided((A.shape[0], col), (ld, 1))


def edgeconv_forward(g: DeviceGraph, H, Theta, Phi):
    """EdgeConv layer forward, reorganized: Y = H [Theta | Phi] (one GEMM),
    then the fused max region.  Theta / Phi given as adjacent column blocks of one buffer
    (EdgeConvNet's parameters) are used in place; separate tensors are concatenated."""
    H = _f32(H, "H")
    if Theta.shape != Phi.shape or Theta.shape[0] != H.shape[1]:
        raise TensorError("edgeconv_forward: Theta/Phi must both be (F_in, C)")
    Wcat = _adjacent_columns([Theta, Phi], "edgeconv_forward")
    if Wcat is None:
        Wcat = torch.cat([_f32(Theta, "Theta"), _f32(Phi, "Phi")], dim=1)
    return edgeconv_forward_cat(g, H, Wcat)


def edgeconv_forward_cat(g: DeviceGraph, H, Wcat):
    """edgeconv_forward on the concatenated weight [Theta | Phi] (F_in x 2C)."""
    C_ = Wcat.shape[1] // 2
    Y = gemm(H, Wcat, ws=g.ws)
    out, amax = edgeconv_region_forward(g, Y[:, :C_], Y[:, C_:])
    return out, EdgeConvStash(Y, amax)


def edgeconv_backward(g: DeviceGraph, H, Theta, Phi, stash: EdgeConvStash, dOut, need_dH=True):
    """Argmax routing (K7) then dY -> d[Theta|Phi] = H^T dY, dH = dY [Theta|Phi]^T.
    Returns (dH, dTheta, dPhi); dTheta / dPhi are column views of one d[Theta|Phi] buffer."""
    Wcat = _adjacent_columns([Theta, Phi], "edgeconv_backward")
    if Wcat is None:
        Wcat = torch.cat([_f32(Theta, "Theta"), _f32(Phi, "Phi")], dim=1)
    dH, dWcat = edgeconv_backward_cat(g, H, Wcat, stash, dOut, need_dH)
    C_ = Theta.shape[1]
    return dH, dWcat[:, :C_], dWcat[:, C_:]


def edgeconv_backward_cat(g: DeviceGraph, H, Wcat, stash: EdgeConvStash, dOut, need_dH=True):
    """(dH, d[Theta|Phi]) of edgeconv_forward_cat."""
    H = _f32(H, "H")
    C_ = Wcat.shape[1] // 2
    dOut = _f32(dOut, "dOut")
    V = g.num_vertices
    dY = torch.empty(V, 2 * C_, device=H.device)
    with PROBE("edgeconv_bwd"):
        call("gnncg_edgeconv_bwd", g.csc_src.struct(), g.csr_dst.struct(), C_, _ptr(stash.argmax), _ptr(dOut),
             _ptr(dY), dY.stride(0), _ptr(dY) + 4 * C_, dY.stride(0), _stream())
    dWcat = gemm(H, dY, trans_a=True, ws=g.ws)
    dH = gemm(dY, Wcat, trans_b=True, ws=g.ws) if need_dH else None
    return dH, dWcat


# ---------------------------------------------------------------------------
# GMMConv
# ---------------------------------------------------------------------------
@dataclass
class GmmStash:
    Y: torch.Tensor  # [hW | pl | pr], V x (K f + 2 r)


def gmm_weight_width(K: int, r: int, f: int) -> int:
    """Row width of [W | P_l | P_r]: K f + 2 r padded to a multiple of 4 floats, so Y and dY
    have 16-byte rows (the TMA tensor-core GEMM needs them; K8 takes ldy >= K f + 2 r)."""
    return (K * f + 2 * r + 3) // 4 * 4


def _gmm_wcat(W, P_l, P_r):
    """[W | P_l | P_r] as one padded matrix: the buffer itself when the three are adjacent
    column blocks of it (MoNet's parameters), else a zero-padded copy (the reference API
    with separate tensors)."""
    n = W.shape[1] + P_l.shape[1] + P_r.shape[1]
    cat = _adjacent_columns([W, P_l, P_r], "gmm")
    if cat is not None and W.stride(0) == (n + 3) // 4 * 4:
        return cat.as_strided((W.shape[0], W.stride(0)), (W.stride(0), 1))
    out = torch.zeros(W.shape[0], (n + 3) // 4 * 4, device=W.device)
    a, b = W.shape[1], W.shape[1] + P_l.shape[1]
    out[:, :a] = _f32(W, "W")
    out[:, a:b] = _f32(P_l, "P_l")
    out[:, b:n] = _f32(P_r, "P_r")
    return out


def gmm_forward(g: DeviceGraph, H, W, P_l, P_r, mu, sinv, K: int, r: int, f: int):
    """GMMConv layer forward: Y = H [W | P_l | P_r], then the fused
    Gaussian-weighted aggregation (K8)."""
    H = _f32(H, "H")
    Fin = H.shape[1]
    _shape(W, (Fin, K * f), "W")
    _shape(P_l, (Fin, r), "P_l")
    _shape(P_r, (Fin, r), "P_r")
    _shape(mu, (K, r), "mu")
    _shape(sinv, (K, r), "sinv")
    Y = gemm(H, _gmm_wcat(W, P_l, P_r), ws=g.ws)
    out = torch.empty(g.num_vertices, f, device=H.device)
    with PROBE("gmm_fwd"):
        call("gnncg_gmm_fwd", g.csr_dst.struct(), K, r, f, _ptr(Y), Y.stride(0), _ptr(_f32(mu, "mu")),
             _ptr(_f32(sinv, "sinv")), _ptr(out), _stream())
    return out, GmmStash(Y)


def gmm_backward(g: DeviceGraph, H, W, P_l, P_r, mu, sinv, K, r, f, stash: GmmStash, dOut, need_dH=True):
    """Returns (dH, dW, dP_l, dP_r, dmu, dsinv); dW / dP_l / dP_r are column views of one
    d[W | P_l | P_r] buffer (padding columns zero), which is returned as the 7th item."""
    H = _f32(H, "H")
    dOut = _f32(dOut, "dOut")
    Y = stash.Y
    dY = torch.empty_like(Y)  # K8 writes every column, the alignment padding as zeros
    dmu = torch.empty(K, r, device=H.device)
    dsinv = torch.empty(K, r, device=H.device)
    need = _lib.lib().gnncg_gmm_bwd_workspace(g.csr_dst.struct(), K, r)
    wp, wn = g.ws.get(need)
    with PROBE("gmm_bwd"):
        call("gnncg_gmm_bwd", g.csr_dst.struct(), g.csc_src.struct(), K, r, f, _ptr(Y), Y.stride(0), _ptr(mu),
             _ptr(sinv), _ptr(dOut), _ptr(dY), _ptr(dmu), _ptr(dsinv), wp, wn, _stream())
    dWcat = gemm(H, dY, trans_a=True, ws=g.ws)
    dH = gemm(dY, _gmm_wcat(W, P_l, P_r), trans_b=True, ws=g.ws) if need_dH else None
    Kf = K * f
    return dH, dWcat[:, :Kf], dWcat[:, Kf:Kf + r], dWcat[:, Kf + r:Kf + 2 * r], dmu, dsinv, dWcat


# ---------------------------------------------------------------------------
# GCN (weighted Aggregate)
# ---------------------------------------------------------------------------
@dataclass
class GcnStash:
    Ht: torch.Tensor  # H W, V x F_out
    out: torch.Tensor  # act(b + A_w Ht)


def gcn_norm(g: DeviceGraph) -> torch.Tensor:
    """Symmetric normalisation by edge id: w[e] = 1/sqrt(max(1,deg_in(dst)) max(1,deg_out(src)))."""
    w = torch.empty(g.num_edges, dtype=torch.float32, device=g.device)
    call("gnncg_gcn_norm", g.num_edges, _ptr(g.edge_src), _ptr(g.edge_dst), g.csr_dst.struct(), g.csc_src.struct(),
         _ptr(w), _stream())
    return w


def spmm(g: DeviceGraph, X, edge_w=None, bias=None, relu=False, transpose=False, out=None, chunk=None):
    """Y = act(bias + A_w X) with A_w[v,u] = sum of w[e] over edges u -> v (transpose: A_w^T X,
    i.e. the sum runs over out-edges).  One fused kernel (csrc/spmm.cu)."""
    X = _f32(X, "X")
    idx = g.csc_src if transpose else g.csr_dst
    V, C_ = g.num_vertices, X.shape[1]
    _shape(X, (V, C_), "X")
    if edge_w is not None:
        edge_w = _f32(edge_w, "edge_w")
        _shape(edge_w, (g.num_edges,), "edge_w")
    if bias is not None:
        bias = _f32(bias, "bias")
        _shape(bias, (C_,), "bias")
    out = torch.empty(V, C_, device=X.device) if out is None else out
    sched = idx.sched(chunk) if chunk else idx.sched()
    need = _lib.lib().gnncg_spmm_workspace(sched.struct(), C_)
    wp, wn = g.ws.get(need)
    with PROBE("spmm_t" if transpose else "spmm"):
        call("gnncg_spmm", idx.struct(), sched.struct(), C_, _ptr(edge_w), _ptr(X), _ptr(bias), int(relu), _ptr(out),
             wp, wn, _stream())
    return out


def gcn_forward(g: DeviceGraph, H, W, b, edge_w=None, relu=True, chunk=None):
    """GCN layer forward: out = relu(b + A_w (H W))  (SPEC.md:184 gcn).
    Transform first (F_out <= F_in on the benchmark shapes), then one fused aggregate kernel."""
    H, W = _f32(H, "H"), _f32(W, "W")
    if W.shape[0] != H.shape[1]:
        raise TensorError("gcn_forward: W must be (F_in, F_out)")
    Ht = gemm(H, W, ws=g.ws)
    out = spmm(g, Ht, edge_w, b, relu, chunk=chunk)
    return out, GcnStash(Ht, out)


def gcn_backward(g: DeviceGraph, H, W, stash: GcnStash, dOut, edge_w=None, relu=True, need_dH=True, chunk=None):
    """Returns (dH, dW, db): dZ = dOut * relu'(out), db = colsum dZ, dHt = A_w^T dZ (csc_src),
    dW = H^T dHt, dH = dHt W^T."""
    H = _f32(H, "H")
    dOut = _f32(dOut, "dOut")
    V, C_ = stash.out.shape
    _shape(dOut, (V, C_), "dOut")
    dZ = torch.empty(V, C_, device=H.device)
    db = torch.empty(C_, device=H.device)
    need = _lib.lib().gnncg_relu_bwd_workspace(C_)
    wp, wn = g.ws.get(need)
    with PROBE("relu_bwd"):
        call("gnncg_relu_bwd", V, C_, _ptr(dOut), _ptr(stash.out), int(relu), _ptr(dZ), _ptr(db), wp, wn, _stream())
    dHt = spmm(g, dZ, edge_w, transpose=True, chunk=chunk)
    dW = gemm(H, dHt, trans_a=True, ws=g.ws)
    dH = gemm(dHt, W, trans_b=True, ws=g.ws) if need_dH else None
    return dH, dW, db
