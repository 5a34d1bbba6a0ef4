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
