"""Alg. 1 rollout driver over the B200 PBSA path, with JSONL memory traces.

Reference: SPEC.md:419-508 (module rollout) and PAPER.md:197-230 (Algorithm 1).  This is the
CALLER of the hot path: it drives one pbsa.Memory per layer through
M chunks x T denoise steps + the k=0 cache-update pass, exactly the call order that defines the
per-chunk decode latency of BASELINE.json, and records the memory trace of SPEC.md:235 (one JSON
record per (chunk, denoise index): persistent ids, window ids, evicted ids, scores, flags).

The denoiser is SPEC's ToyDenoiser: seeded linear maps W_q, W_k, W_v,
W_o per layer on blockified latents; x_hat_0 = W_o . PBSA output (+ residual).  It is plumbing
(torch matmuls); the attention/memory path is the product (pbsa.Memory -> libpbsa_b200.so).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import time

import torch

from . import pbsa

# ---------------------------------------------------------------- configuration


@dataclasses.dataclass
class RolloutConfig:
    num_chunks: int = 4                      # M
    timesteps: tuple = (1.0, 0.75, 0.5, 0.25)  # t_T .. t_1, strictly decreasing
    topk_ratio: float = 0.25
    capacity_frames: int = 6                 # C
    window_frames: int = 6                   # L_local (frames; whole chunks; SPEC.md:493 default)
    chunk_frames: int = 3
    height: int = 30
    width: int = 52
    block_shape: tuple = (1, 15, 4)          # (b_t, b_h, b_w)
    layers: int = 2
    heads: int = 12
    head_dim: int = 128
    seed: int = 7
    trace_units: int = 1                     # heads recorded in the trace (unit 0..n-1)
    latent: bool = True                      # chunks stay (t, h, w, d) latents (pbsa_attend_latent);
                                             # False: blockify in torch + pbsa_attend_qkv

    def validate(self):
        ts = list(self.timesteps)
        if not ts or any(not (0.0 < t <= 1.0) for t in ts) or any(a <= b for a, b in zip(ts, ts[1:])):
            raise ValueError("timesteps must be strictly decreasing values in (0,1]")
        if self.num_chunks < 1:
            raise ValueError("num_chunks must be >= 1")
        bt, bh, bw = self.block_shape
        for ax, n, bsz in (("t", self.chunk_frames, bt), ("h", self.height, bh), ("w", self.width, bw)):
            if n % bsz:
                raise ValueError(f"axis {ax} ({n}) not divisible by block extent ({bsz})")
        if self.window_frames % self.chunk_frames or self.capacity_frames % bt:
            raise ValueError("window must be whole chunks and capacity whole block rows")

    @property
    def b(self) -> int:
        return self.block_shape[0] * self.block_shape[1] * self.block_shape[2]

    @property
    def blocks_per_frame(self) -> int:
        return (self.height // self.block_shape[1]) * (self.width // self.block_shape[2])

    @property
    def blocks_per_chunk(self) -> int:
        return (self.chunk_frames // self.block_shape[0]) * self.blocks_per_frame

    @property
    def capacity_blocks(self) -> int:
        return (self.capacity_frames // self.block_shape[0]) * self.blocks_per_frame

    @property
    def window_chunks(self) -> int:
        return self.window_frames // self.chunk_frames

    @property
    def d_model(self) -> int:
        return self.heads * self.head_dim


def sigma(t: float) -> float:
    """Linear schedule, sigma(0) = 0."""
    return float(t)


def renoise(x0_hat: torch.Tensor, eps: torch.Tensor, t: float) -> torch.Tensor:
    """Psi(x0_hat, eps, t) = (1 - sigma(t)) x0_hat + sigma(t) eps."""
    if x0_hat.shape != eps.shape:
        raise ValueError("renoise: shape mismatch")
    s = sigma(t)
    return (1.0 - s) * x0_hat + s * eps


def blockify_tokens(x: torch.Tensor, shape) -> torch.Tensor:
    """(t, h, w, d) -> block-major (n_b*b, d) (blockify.cpp:38-65)."""
    t, h, w, d = x.shape
    bt, bh, bw = shape
    x = x.reshape(t // bt, bt, h // bh, bh, w // bw, bw, d).permute(0, 2, 4, 1, 3, 5, 6)
    return x.reshape(-1, d)


def unblockify_tokens(xb: torch.Tensor, dims, shape) -> torch.Tensor:
    t, h, w, d = dims
    bt, bh, bw = shape
    x = xb.reshape(t // bt, h // bh, w // bw, bt, bh, bw, d).permute(0, 3, 1, 4, 2, 5, 6)
    return x.reshape(t, h, w, d)


class ToyDenoiser:
    """Seeded linear maps per layer; deterministic per seed."""

    def __init__(self, cfg: RolloutConfig, device="cuda"):
        g = torch.Generator(device="cpu").manual_seed(cfg.seed)
        dm = cfg.d_model
        std = 1.0 / math.sqrt(dm)
        self.w = [[(torch.randn(dm, dm, generator=g) * std).to(device, torch.bfloat16) for _ in range(4)]
                  for _ in range(cfg.layers)]
        self.cfg = cfg

    def qkv(self, layer: int, x: torch.Tensor, t: float):
        """x: [n_tok, d_model] bf16 (block-major tokens) -> q, k, v as [heads, n_tok, head_dim]."""
        cfg = self.cfg
        wq, wk, wv, _ = self.w[layer]
        # RMS-normalised layer input (keeps a deep toy stack finite) + timestep conditioning
        xf = x.float()
        xt = (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6) * (1.0 + 0.1 * t)).to(x.dtype)
        out = []
        for w in (wq, wk, wv):
            y = (xt @ w).view(x.shape[0], cfg.heads, cfg.head_dim).transpose(0, 1).contiguous()
            out.append(y)
        return out

    def qkv_tokens(self, layer: int, x: torch.Tensor, t: float):
        """x: [n_tok, d_model] bf16 in any token order -> q, k, v [n_tok, heads*head_dim]: for a
        (t, h, w) token order these ARE the Latent4D chunk latents pbsa_attend_latent consumes."""
        wq, wk, wv, _ = self.w[layer]
        xf = x.float()
        xt = (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6) * (1.0 + 0.1 * t)).to(x.dtype)
        return [xt @ w for w in (wq, wk, wv)]

    def project_out_tokens(self, layer: int, o: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        """o: [n_tok, heads*head_dim] -> residual update of x [n_tok, d_model]."""
        return x + (o @ self.w[layer][3]) * (1.0 / self.cfg.layers)

    def project_out(self, layer: int, o: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        """o: [heads, n_tok, head_dim] -> residual update of x."""
        wo = self.w[layer][3]
        y = o.transpose(0, 1).reshape(x.shape[0], self.cfg.d_model) @ wo
        return x + y * (1.0 / self.cfg.layers)


# ---------------------------------------------------------------- Alg. 1


def _per_head(x: torch.Tensor, cfg: RolloutConfig) -> torch.Tensor:
    """Chunk tokens of one layer call -> [heads, bpc*b, head_dim] f32 in block-major token order (the
    per-unit layout of the C ABI), from a (t, h, w, d) latent or an already block-major tensor."""
    if cfg.latent:
        x = blockify_tokens(x.reshape(cfg.chunk_frames, cfg.height, cfg.width, cfg.d_model), cfg.block_shape)
        return x.reshape(-1, cfg.heads, cfg.head_dim).transpose(0, 1).float().cpu()
    return x.float().cpu()


def run_inference(cfg: RolloutConfig, denoiser: ToyDenoiser | None = None, trace_path: str | None = None,
                  device="cuda", record_scores: bool = True, capture: list | None = None):
    """Returns (frames [list of (t,h,w,d) bf16 chunks], trace [list of dicts], timing dict).

    capture (a list): every layer-0 PBSA call appends {"mode", "k_top", "q", "k", "v", "o" (all
    [heads, bpc*b, head_dim] f32, block-major), "sel" [heads, bpc, k] (or None), "s_t" [heads,
    n_keys] (k=0 pass), "persistent" / "window" (ids after the call)} -- the record an oracle replay
     consumes."""
    cfg.validate()
    den = denoiser or ToyDenoiser(cfg, device)
    bpc, b, U = cfg.blocks_per_chunk, cfg.b, cfg.heads
    k_top = None
    mems = [pbsa.Memory(U, cfg.capacity_blocks, cfg.window_chunks, bpc, b, cfg.head_dim)
            for _ in range(cfg.layers)]
    g = torch.Generator(device=device).manual_seed(cfg.seed + 1)
    dims = (cfg.chunk_frames, cfg.height, cfg.width, cfg.d_model)
    frames, trace = [], []
    calls = 0
    stream = torch.cuda.current_stream()
    ev = []
    for i in range(cfg.num_chunks):
        x = torch.randn(dims, device=device, generator=g).to(torch.bfloat16)  # x ~ N(0, I)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        def layer_stack(xin, t, mode, scores_rec=None):
            """All layers of the toy denoiser on one chunk; returns the chunk latent out."""
            nonlocal calls
            dm = cfg.d_model
            h = xin.reshape(-1, dm) if cfg.latent else blockify_tokens(xin, cfg.block_shape)
            for layer, mem in enumerate(mems):
                n_l = mem.info().n_l
                k_top = pbsa.topk_count(n_l, cfg.topk_ratio) if n_l else 0
                if cfg.latent:  # (t, h, w) tokens: blockify / unblockify happen inside the kernels
                    q, k, v = den.qkv_tokens(layer, h, t)
                    o = mem.attend_latent(q.view(dims), k.view(dims), v.view(dims), cfg.block_shape, k_top, mode)
                    h = den.project_out_tokens(layer, o.view(-1, dm), h)
                else:
                    q, k, v = den.qkv(layer, h, t)
                    o = mem.attend_qkv(q, k, v, k_top, mode)
                    h = den.project_out(layer, o, h)
                if scores_rec is not None and layer == 0 and mode == pbsa.MODE_CACHE_UPDATE:
                    _, s_t = mem.last_selection()
                    scores_rec["scores"] = [[float(v_) for v_ in s_t[u].tolist()] for u in range(cfg.trace_units)]
                if capture is not None and layer == 0:
                    sel, s_t = mem.last_selection()
                    p_ids, l_ids = mem.assemble()
                    capture.append({"mode": mode, "k_top": k_top, "q": _per_head(q, cfg), "k": _per_head(k, cfg),
                                    "v": _per_head(v, cfg), "o": _per_head(o, cfg),
                                    "sel": None if sel is None else sel.cpu(),
                                    "s_t": s_t.cpu() if mode == pbsa.MODE_CACHE_UPDATE and s_t is not None else None,
                                    "persistent": p_ids.cpu(), "window": l_ids.cpu()})
                calls += 1
            return h.view(dims) if cfg.latent else unblockify_tokens(h, dims, cfg.block_shape)

        for jj, t in enumerate(cfg.timesteps):
            j = len(cfg.timesteps) - jj  # j = T .. 1
            x0_hat = layer_stack(x, t, pbsa.MODE_DENOISE)
            rec = {"chunk": i, "j": j, "t": t, "cache_updated": j == 1, "grad_enabled": False}
            # every record carries the layer-0 memory it attended over
            p_ids, l_ids = _ids(mems[0], cfg.trace_units)
            rec["persistent"], rec["window"], rec["evicted"] = p_ids, l_ids, [[] for _ in range(cfg.trace_units)]
            if j == 1:
                frames.append(x0_hat)
                # k = 0 pass on the clean chunk: scores, push/evict, Top-C (Alg. 1 lines 9-10)
                layer_stack(x0_hat, 0.0, pbsa.MODE_CACHE_UPDATE, rec if record_scores else None)
                prev_l = l_ids
                p_ids, l_ids = _ids(mems[0], cfg.trace_units)
                rec["evicted"] = [sorted(set(prev_l[u]) - set(l_ids[u])) for u in range(cfg.trace_units)]
                rec["persistent"] = p_ids
                rec["window"] = l_ids
            else:
                eps = torch.randn(dims, device=device, generator=g).to(torch.bfloat16)
                x = renoise(x0_hat, eps, cfg.timesteps[jj + 1]).to(torch.bfloat16)
            trace.append(rec)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    chunk_ms = [a.elapsed_time(b_) for a, b_ in ev]
    status = max(m.status() for m in mems)
    for m in mems:
        m.close()
    if trace_path:
        with open(trace_path, "w") as f:
            for rec in trace:
                f.write(json.dumps(rec) + "\n")
    return frames, trace, {"chunk_ms": chunk_ms, "pbsa_calls": calls, "invalid_input_flags": status}


def _ids(mem: pbsa.Memory, n_units: int):
    p, l_ = mem.assemble()
    return [p[u].tolist() for u in range(n_units)], [l_[u].tolist() for u in range(n_units)]


def check_trace(cfg: RolloutConfig, trace) -> None:
    """SPEC.md:484-488 / acceptance 6: cache updates exactly once per chunk at j=1, |P| <= C and
    |window| <= L_local at every record, P and L disjoint, evicted ids strictly increasing, and the
    sinks (blocks of the first chunk) retained once they entered P -- for every traced
    unit."""
    updates = [r for r in trace if r["cache_updated"]]
    if len(updates) != cfg.num_chunks or any(r["j"] != 1 for r in updates):
        raise AssertionError("cache updates must happen exactly once per chunk, at j = 1")
    if len(trace) != cfg.num_chunks * len(cfg.timesteps):
        raise AssertionError("one trace record per (chunk, denoise step)")
    n_units = len(trace[0]["persistent"]) if trace else 0
    for r in trace:
        for p, l_ in zip(r["persistent"], r["window"]):
            if len(p) > cfg.capacity_blocks or len(l_) > cfg.window_chunks * cfg.blocks_per_chunk:
                raise AssertionError("capacity exceeded")
            if set(p) & set(l_):
                raise AssertionError("P and L overlap")
    sinks = set(range(cfg.blocks_per_chunk))
    for u in range(n_units):
        last, sunk = -1, False
        for r in updates:
            ev = r["evicted"][u]
            if ev:
                if min(ev) <= last:
                    raise AssertionError("eviction ids must strictly increase")
                last = max(ev)
            p = set(r["persistent"][u])
            if sunk and not sinks <= p:
                raise AssertionError(f"sink retention violated (unit {u}, chunk {r['chunk']})")
            sunk = sunk or sinks <= p


def main(argv=None):
    ap = argparse.ArgumentParser(description="Sparse Forcing Alg. 1 rollout on the B200 PBSA path")
    ap.add_argument("--frames", type=int, default=12, help="latent frames to generate (multiple of chunk)")
    ap.add_argument("--steps", type=int, default=4, help="denoise steps T")
    ap.add_argument("--topk", type=float, default=0.25)
    ap.add_argument("--capacity-frames", type=int, default=6)
    ap.add_argument("--window-frames", type=int, default=6)
    ap.add_argument("--layers", type=int, default=30)
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    if a.frames < 3 or a.frames % 3:
        raise SystemExit(2)
    ts = tuple(1.0 - i / a.steps for i in range(a.steps))
    cfg = RolloutConfig(num_chunks=a.frames // 3, timesteps=ts, topk_ratio=a.topk,
                        capacity_frames=a.capacity_frames, window_frames=a.window_frames,
                        layers=a.layers, heads=a.heads, seed=a.seed)
    trace_path = None
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        trace_path = os.path.join(a.out, "trace.jsonl")
    t0 = time.time()
    frames, trace, timing = run_inference(cfg, trace_path=trace_path)
    check_trace(cfg, trace)
    if a.out:  # frames as PBT1 tensors, Latent4D (t, h, w, d) f32
        for i, fr in enumerate(frames):
            pbsa.write_tensor(os.path.join(a.out, f"frame_{i:04d}.pbt1"), fr.float().cpu().numpy())
    steady = timing["chunk_ms"][cfg.window_chunks + 2:] or timing["chunk_ms"]
    print(json.dumps({"chunks": cfg.num_chunks, "layers": cfg.layers, "heads": cfg.heads,
                      "pbsa_calls": timing["pbsa_calls"], "chunk_ms": timing["chunk_ms"],
                      "invalid_input_flags": timing["invalid_input_flags"],
                      "steady_chunk_ms_median": sorted(steady)[len(steady) // 2],
                      "wall_s": time.time() - t0}))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
