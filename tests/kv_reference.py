"""fp32 reference for the N2/N3 data plane: the synthetic KV content and
decode queries of csrc/data_plane.cuh restated in numpy, and the decode
attention softmax(q K^T / sqrt(d)) V computed from them."""
import numpy as np

M32 = 0xFFFFFFFF


def _mix32(h):
    h = h & M32
    h ^= h >> 16
    h = (h * 0x7FEB352D) & M32
    h ^= h >> 15
    h = (h * 0x846CA68B) & M32
    h ^= h >> 16
    return h


def kv_values(rid, toks, row, dims):
    """bf16-exact KV values for tokens x dims of one row, as float32."""
    t = np.asarray(toks, dtype=np.uint64)[:, None]
    d = np.asarray(dims, dtype=np.uint64)[None, :]
    inner = _mix32((t * 0x85EBCA77 + np.uint64(row) * 0xC2B2AE3D + d * 0x27D4EB2F) & M32)
    h = _mix32((np.uint64(rid) * 0x9E3779B1 & M32) ^ inner)
    return ((h >> 24).astype(np.uint8).view(np.int8).astype(np.float32)) / 128.0


def q_values(rid, step, layer, qh, dims):
    d = np.asarray(dims, dtype=np.uint64)
    inner = _mix32((np.uint64(step) * 0x9E3779B9 + np.uint64(layer) * 0x632BE5AB + np.uint64(qh) * 0x85157AF5
                    + d * 0x4CF5AD43) & M32)
    h = _mix32((np.uint64(rid) * 0x2545F491 & M32) ^ inner)
    return (h >> 20).astype(np.float32) / 2048.0 - 1.0


def decode_reference(rid, ctx, step, layers, hq, hkv, dim=128):
    """out[layer][q_head][dim] fp32 for one decode member."""
    g = hq // hkv
    out = np.zeros((layers, hq, dim), dtype=np.float64)
    toks = np.arange(ctx)
    dims = np.arange(dim)
    for layer in range(layers):
        for kh in range(hkv):
            K = kv_values(rid, toks, (layer * 2 + 0) * hkv + kh, dims).astype(np.float64)
            V = kv_values(rid, toks, (layer * 2 + 1) * hkv + kh, dims).astype(np.float64)
            for j in range(g):
                qh = kh * g + j
                q = q_values(rid, step, layer, qh, dims).astype(np.float64)
                s = K @ q / np.sqrt(dim)
                p = np.exp(s - s.max())
                out[layer, qh] = (p / p.sum()) @ V
    return out


# -- the same reference on a torch device (int64 hashing + float64 attention),
# so full-size layouts (Llama-2-70B: 80 layers x 8 KV heads) check in seconds

def _mix32_t(h):
    M = 0xFFFFFFFF
    h = h & M
    h = h ^ (h >> 16)
    h = (h * 0x7FEB352D) & M
    h = h ^ (h >> 15)
    h = (h * 0x846CA68B) & M  # int64 wrap-around keeps the low 32 bits exact
    h = h ^ (h >> 16)
    return h


def decode_reference_torch(rid, ctx, step, layers, hq, hkv, dim=128, device="cuda"):
    """decode_reference() evaluated with torch on `device`; returns numpy
    float64 out[layer][q_head][dim]."""
    import torch
    M = 0xFFFFFFFF
    g = hq // hkv
    i64 = dict(dtype=torch.int64, device=device)
    t = torch.arange(ctx, **i64)[:, None]
    d = torch.arange(dim, **i64)
    rows = torch.arange(layers * 2 * hkv, **i64)
    inner = _mix32_t((t[None] * 0x85EBCA77 + rows[:, None, None] * 0xC2B2AE3D + d[None, None] * 0x27D4EB2F) & M)
    h = _mix32_t(((rid * 0x9E3779B1) & M) ^ inner)
    b = (h >> 24) & 0xFF
    kv = torch.where(b >= 128, b - 256, b).to(torch.float64) / 128.0      # [rows, ctx, dim]
    kv = kv.view(layers, 2, hkv, ctx, dim)
    K, V = kv[:, 0], kv[:, 1]                                             # [L, hkv, ctx, dim]
    lay = torch.arange(layers, **i64)[:, None, None]
    qh = torch.arange(hq, **i64)[None, :, None]
    qi = _mix32_t((step * 0x9E3779B9 + lay * 0x632BE5AB + qh * 0x85157AF5 + d[None, None] * 0x4CF5AD43) & M)
    q = ((_mix32_t(((rid * 0x2545F491) & M) ^ qi) >> 20).to(torch.float64) / 2048.0 - 1.0)   # [L, hq, dim]
    q = q.view(layers, hkv, g, dim)
    s = torch.einsum("lkgd,lkcd->lkgc", q, K) / (dim ** 0.5)
    p = torch.softmax(s, dim=-1)
    out = torch.einsum("lkgc,lkcd->lkgd", p, V).reshape(layers, hq, dim)
    return out.cpu().numpy()
