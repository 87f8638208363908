"""Fetch-codec microbenchmark: encode one expert-sized bf16 buffer, then time
the decoder (whole blob and per piece, CUDA events, warm) and a pinned
host -> device copy of the coded vs raw bytes.

    python tools/xfer_bench.py [--values 176160768] [--iters 20]

Prints one JSON line: coded/raw ratio, decode GB/s (read coded + write
bf16 over kernel time), per-piece decode us, H2D ms raw vs coded.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_10054_b200 import _native as N  # noqa: E402
from paper_2511_10054_b200 import ops  # noqa: E402


def _time(fn, iters):
    evs = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--values", type=int, default=3 * 4096 * 14336)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--format", type=int, default=0, help="piece format 2 or 3 (0: the library default)")
    args = ap.parse_args()
    if args.format:
        os.environ["BMOE_XFER_FORMAT"] = str(args.format)
    n = args.values
    x = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    x[: 2 * n // 3].normal_(0.0, 4096 ** -0.5)
    x[2 * n // 3:].normal_(0.0, 14336 ** -0.5)
    blob = ops.xfer_encode(x)
    y = torch.empty_like(x)
    ms_blob = _time(lambda: ops.xfer_decode(blob, n, y), args.iters)
    assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    # the first and the last piece alone, as the engine decodes them from the staging ring
    hb = blob[:256].cpu().numpy()
    n_pieces = int(np.frombuffer(hb[4:8].tobytes(), np.uint32)[0])
    pv = int(np.frombuffer(hb[16:20].tobytes(), np.uint32)[0])
    offs = [int(v) for v in np.frombuffer(blob[24:24 + 8 * (n_pieces + 1)].cpu().numpy().tobytes(), np.uint64)]
    s = torch.cuda.current_stream().cuda_stream
    pieces = {}
    for name, p in (("first", 0), ("last", n_pieces - 1)):
        piece = blob[offs[p]:offs[p + 1]]
        nch = int(np.frombuffer(piece[4:8].cpu().numpy().tobytes(), np.uint32)[0])
        nv = min(pv, n - p * pv)
        ms = _time(lambda: N.call("bm_xfer_decode_piece", piece.data_ptr(), y[p * pv:].data_ptr(), nch, s),
                   args.iters)
        pieces[name] = {"values": nv, "us": ms * 1e3, "gbs": (offs[p + 1] - offs[p] + 2 * nv) / ms / 1e6}
    assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    magic = int(np.frombuffer(blob[offs[0]:offs[0] + 4].cpu().numpy().tobytes(), np.uint32)[0])
    # pinned H2D of the coded vs raw bytes
    hraw = torch.empty(2 * n, dtype=torch.uint8).pin_memory()
    hcod = torch.empty(blob.numel(), dtype=torch.uint8).pin_memory()
    draw = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    ms_raw = _time(lambda: draw.copy_(hraw, non_blocking=True), 5)
    ms_cod = _time(lambda: draw[: blob.numel()].copy_(hcod, non_blocking=True), 5)
    moved = blob.numel() + 2 * n
    out = {"values": n, "coded_bytes": blob.numel(), "ratio": blob.numel() / (2 * n),
           "decode_ms": ms_blob, "decode_gbs": moved / ms_blob / 1e6, "decode_out_gbs": 2 * n / ms_blob / 1e6,
           "piece_format": {0x32505842: 2, 0x33505842: 3}.get(magic, magic), "pieces": pieces,
           "h2d_raw_ms": ms_raw, "h2d_coded_ms": ms_cod, "h2d_gbs": 2 * n / ms_raw / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
