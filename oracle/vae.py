"""VAE decoder: whole-image decode and the V1 chunked decode (ORACLE — test infrastructure only).

Paper: "VAE Chunking partitions the decoder into N temporally equivalent sub-blocks at the
ResNet block level" (§III-B; fig:mot3 PAPER.md:165-172). North star: "the
latent is split into halo-padded tiles, decoded tile by tile and stitched".

Reading R7, "V1 stage-synchronous halo tiles", is what `decode_chunked`
implements, as a separate code path from `decode`:
  * head items (post_quant_conv, conv_in, mid block incl. the global attention) run on the
    whole latent;
  * every later layer is cut into row bands; a conv band reads its input band plus a
    `halo`-row halo (zero outside the image = the conv's padding) and writes a disjoint band
    of the full output (stitching = disjoint writes);
  * GroupNorm statistics are per-band partials (count, mean, M2) merged in fixed band order
    (Chan et al.), then applied band by band;
  * the ordered item list is cut into `c` contiguous chunks (`chunk_ranges`).
Invariant I6: decode_chunked == decode for any c / band count (fp64 ≤ 1e-12); halo 0 must fail.
"""
from __future__ import annotations

import numpy as np

from . import nn
from .configs import VAEConfig, vae_structure
from .unet import resnet as _resnet


def _vae_attention(P, p, x, groups, eps):
    N, C, H, W = x.shape
    h = nn.group_norm(x, groups, P[p + ".group_norm.weight"], P[p + ".group_norm.bias"], eps)
    h = h.reshape(N, C, H * W).transpose(0, 2, 1)
    q = nn.linear(h, P[p + ".to_q.weight"], P[p + ".to_q.bias"])
    k = nn.linear(h, P[p + ".to_k.weight"], P[p + ".to_k.bias"])
    v = nn.linear(h, P[p + ".to_v.weight"], P[p + ".to_v.bias"])
    o = nn.attention(q, k, v)                                   # 1 head, d = C (R28)
    o = nn.linear(o, P[p + ".to_out.0.weight"], P[p + ".to_out.0.bias"])
    return o.transpose(0, 2, 1).reshape(N, C, H, W) + x


def head(P, cfg: VAEConfig, z):
    """z/σ_vae → post_quant_conv → conv_in → mid (res, attention, res)."""
    g, e = cfg.groups, cfg.eps
    h = z / z.dtype.type(cfg.scaling_factor)
    h = nn.conv2d(h, P["post_quant_conv.weight"], P["post_quant_conv.bias"], pad=0)
    h = nn.conv2d(h, P["decoder.conv_in.weight"], P["decoder.conv_in.bias"])
    h = _resnet(P, "decoder.mid_block.resnets.0", h, None, g, e)
    h = _vae_attention(P, "decoder.mid_block.attentions.0", h, g, e)
    return _resnet(P, "decoder.mid_block.resnets.1", h, None, g, e)


def decode(P, cfg: VAEConfig, z):
    """Whole-image decode. z [N,4,h,w] → image [N,3,8h·…] (float, before clamp; R23)."""
    g, e = cfg.groups, cfg.eps
    h = head(P, cfg, z)
    for i, blk in enumerate(vae_structure(cfg)):
        for j in range(len(blk["res"])):
            h = _resnet(P, f"decoder.up_blocks.{i}.resnets.{j}", h, None, g, e)
        if blk["up"]:
            h = nn.upsample_nearest2x(h)
            h = nn.conv2d(h, P[f"decoder.up_blocks.{i}.upsamplers.0.conv.weight"],
                          P[f"decoder.up_blocks.{i}.upsamplers.0.conv.bias"])
    h = nn.silu(nn.group_norm(h, g, P["decoder.conv_norm_out.weight"], P["decoder.conv_norm_out.bias"], e))
    return nn.conv2d(h, P["decoder.conv_out.weight"], P["decoder.conv_out.bias"])


# ---------------------------------------------------------------------------------------------
# V1 chunked decode (R7) — separate code path
# ---------------------------------------------------------------------------------------------

def _bands(H, n_bands):
    n = max(1, min(n_bands, H))
    edges = [(H * k) // n for k in range(n + 1)]
    return [(edges[k], edges[k + 1]) for k in range(n)]


def work_items(cfg: VAEConfig, h, w, n_bands):
    """Ordered decode work list [(op, args)]; tail ops carry a band (y0, y1)."""
    items = [("head", {})]
    R = h                                                       # current spatial height
    C = cfg.block_out[-1]
    cur = "x"
    nb = 0

    def gn(src, dst, name, silu):
        for bd in _bands(R, n_bands):
            items.append(("gn_stats", dict(src=src, name=name, band=bd)))
        for bd in _bands(R, n_bands):
            items.append(("gn_apply", dict(src=src, dst=dst, name=name, silu=silu, band=bd)))

    def conv(src, dst, wname, up=False, res=None, pad=1):
        RR = 2 * R if up else R
        for bd in _bands(RR, n_bands):
            items.append(("conv", dict(src=src, dst=dst, w=wname, band=bd, up=up, res=res, pad=pad)))

    for i, blk in enumerate(vae_structure(cfg)):
        for j, (ci, co) in enumerate(blk["res"]):
            p = f"decoder.up_blocks.{i}.resnets.{j}"
            nb += 1
            gn(cur, "t1", p + ".norm1", True)
            conv("t1", "t2", p + ".conv1")
            gn("t2", "t1", p + ".norm2", True)
            if ci != co:
                conv(cur, "t3", p + ".conv_shortcut", pad=0)
                conv("t1", "y", p + ".conv2", res="t3")
            else:
                conv("t1", "y", p + ".conv2", res=cur)
            items.append(("swap", dict(a="y", b=cur)))
            C = co
        if blk["up"]:
            conv(cur, "y", f"decoder.up_blocks.{i}.upsamplers.0.conv", up=True)
            items.append(("swap", dict(a="y", b=cur)))
            R *= 2
    gn(cur, "t1", "decoder.conv_norm_out", True)
    conv("t1", "img", "decoder.conv_out")
    return items


def chunk_ranges(costs, c):
    """Cut the ordered item list into c non-empty contiguous ranges minimising the maximum chunk
    cost (integer costs, R7 "min-max partition … ties cut earlier"): cap = the optimal maximum;
    then every boundary is placed at the earliest position from which the rest still fits in the
    remaining chunks under cap. Returns boundaries [0 = w_0 < w_1 < … < w_c = len(costs)]."""
    n = len(costs)
    c = max(1, min(int(c), n))
    pre = [0]
    for x in costs:
        pre.append(pre[-1] + int(x))

    def need(s, cap):                      # greedy number of chunks for items [s, n)
        if s >= n:
            return 0
        cnt, start = 1, s
        for k in range(s + 1, n + 1):
            if pre[k] - pre[start] > cap:
                start, cnt = k - 1, cnt + 1
        return cnt

    lo, hi = max(int(x) for x in costs), pre[-1]
    while lo < hi:
        mid = (lo + hi) // 2
        if need(0, mid) <= c:
            hi = mid
        else:
            lo = mid + 1
    cap = lo
    bounds = [0]
    for j in range(1, c):
        s = bounds[-1]
        e = s + 1
        while not (pre[e] - pre[s] <= cap and need(e, cap) <= c - j and n - e >= c - j):
            e += 1
        bounds.append(e)
    bounds.append(n)
    return bounds


def _slab(x, y0, y1, halo, up):
    """Input slab for output rows [y0,y1): rows y0-halo … y1-1+halo of the (optionally 2×-upsampled)
    input, zero outside the image, zero-padded by 1 column on each side."""
    N, C, H, W = x.shape
    HH, WW = (2 * H, 2 * W) if up else (H, W)
    rows = y1 - y0 + 2
    s = np.zeros((N, C, rows, WW + 2), dtype=x.dtype)
    for r in range(rows):
        yy = y0 - 1 + r
        if yy < 0 or yy >= HH:
            continue
        if (r == 0 or r == rows - 1) and halo == 0:
            continue                                            # negative control: no halo
        src = x[:, :, yy // 2 if up else yy, :]
        s[:, :, r, 1:WW + 1] = src.repeat(2, axis=-1) if up else src
    return s


def decode_chunked(P, cfg: VAEConfig, z, n_chunks=2, n_bands=4, halo=1, costs=None, trace=None):
    """V1 chunked decode. Runs the item list in `n_chunks` contiguous ranges (each range would be
    one concurrent round on the GPU). Result must equal `decode` (I6)."""
    g, e = cfg.groups, cfg.eps
    N, _, h, w = z.shape
    items = work_items(cfg, h, w, n_bands)
    if costs is None:
        costs = [1] * len(items)
    bounds = chunk_ranges(costs, n_chunks)
    buf = {}
    parts = {}
    for ci in range(len(bounds) - 1):
        for op, a in items[bounds[ci]:bounds[ci + 1]]:
            if trace is not None:
                trace.append((ci, op))
            if op == "head":
                buf["x"] = head(P, cfg, z)
            elif op == "swap":
                buf[a["b"]] = buf.pop(a["a"])
            elif op == "gn_stats":
                x = buf[a["src"]]
                y0, y1 = a["band"]
                xs = x[:, :, y0:y1, :]
                Nn, C = xs.shape[:2]
                xg = xs.reshape(Nn, g, C // g, -1).reshape(Nn, g, -1)
                cnt = xg.shape[2]
                mean = xg.mean(axis=2)
                m2 = ((xg - mean[:, :, None]) ** 2).sum(axis=2)
                parts.setdefault((a["name"], a["src"]), []).append((cnt, mean, m2))
            elif op == "gn_apply":
                x = buf[a["src"]]
                key = (a["name"], a["src"])
                plist = parts[key]
                n_, mean, m2 = plist[0]
                for (nb_, mb, m2b) in plist[1:]:                 # Chan merge, fixed band order
                    tot = n_ + nb_
                    d = mb - mean
                    mean = mean + d * (nb_ / tot)
                    m2 = m2 + m2b + d * d * (n_ * nb_ / tot)
                    n_ = tot
                var = m2 / n_
                y0, y1 = a["band"]
                if a["dst"] not in buf or buf[a["dst"]].shape != x.shape:
                    buf[a["dst"]] = np.zeros_like(x)
                xs = x[:, :, y0:y1, :]
                Nn, C = xs.shape[:2]
                xg = xs.reshape(Nn, g, -1)
                yv = ((xg - mean[:, :, None]) / np.sqrt(var[:, :, None] + e)).reshape(xs.shape)
                yv = yv * P[a["name"] + ".weight"].reshape(1, C, 1, 1) + P[a["name"] + ".bias"].reshape(1, C, 1, 1)
                if a["silu"]:
                    yv = nn.silu(yv)
                buf[a["dst"]][:, :, y0:y1, :] = yv
                if a is not None and y1 == x.shape[2]:
                    parts.pop(key)
            elif op == "conv":
                x = buf[a["src"]]
                wt = P[a["w"] + ".weight"]
                bs = P[a["w"] + ".bias"]
                y0, y1 = a["band"]
                Nn, C, H, W = x.shape
                HH, WW = (2 * H, 2 * W) if a["up"] else (H, W)
                O = wt.shape[0]
                if a["dst"] not in buf or buf[a["dst"]].shape != (Nn, O, HH, WW):
                    buf[a["dst"]] = np.zeros((Nn, O, HH, WW), dtype=x.dtype)
                if a["pad"] == 0:                                # 1×1 shortcut: no halo needed
                    out = nn.conv2d(x[:, :, y0:y1, :], wt, bs, pad=0)
                else:
                    s = _slab(x, y0, y1, halo, a["up"])
                    out = nn.conv2d(s, wt, bs, pad=0)
                if a["res"] is not None:
                    out = out + buf[a["res"]][:, :, y0:y1, :]
                buf[a["dst"]][:, :, y0:y1, :] = out
    return buf["img"]


# ---------------------------------------------------------------------------------------------
# V2 independent-tile decode — an approximation, separate code path
# ---------------------------------------------------------------------------------------------

def tile_windows(h, w, tile, halo):
    """The tiles of a V2 decode in row-major order: (y0, y1, x0, x1) latent rows / columns the tile
    owns, and (a0, a1, b0, b1) the halo-padded window it is decoded from (clipped at the border)."""
    out = []
    for y0 in range(0, h, tile):
        for x0 in range(0, w, tile):
            y1, x1 = min(h, y0 + tile), min(w, x0 + tile)
            out.append(((y0, y1, x0, x1), (max(0, y0 - halo), min(h, y1 + halo), max(0, x0 - halo), min(w, x1 + halo))))
    return out


def decode_tiled(P, cfg: VAEConfig, z, tile, halo):
    """Reading V2 of R7: the north star's literal "latent split into halo-padded tiles, decoded tile
    by tile and stitched". Every `tile`×`tile` block of latent pixels is decoded ON ITS OWN from its
    `halo`-padded window — GroupNorm statistics and the mid-block attention see only that window, so
    unlike V1 this approximates decode() — and the block's own image region (upscale× its latent
    extent) is cut out of the window's decode and written into the output (stitching = disjoint
    writes, no blending). tile ≥ image, or halo ≥ image, reduces to decode() exactly."""
    N, _, h, w = z.shape
    f = 2 ** (len(cfg.block_out) - 1)
    out = None
    for (y0, y1, x0, x1), (a0, a1, b0, b1) in tile_windows(h, w, tile, halo):
        img = decode(P, cfg, np.ascontiguousarray(z[:, :, a0:a1, b0:b1]))
        if out is None:
            out = np.zeros((N, img.shape[1], f * h, f * w), img.dtype)
        out[:, :, f * y0:f * y1, f * x0:f * x1] = img[:, :, f * (y0 - a0):f * (y1 - a0), f * (x0 - b0):f * (x1 - b0)]
    return out
