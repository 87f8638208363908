"""Pinned host -> HBM copy bandwidth (the fetch roofline of an expert miss).
Copies one Mixtral expert (352,321,536 B) from pinned memory with 1 or 2
streams and several chunkings; prints GB/s per variant as JSON."""

import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_10054_b200 import _native as N  # noqa: E402
from paper_2511_10054_b200.engine import HostMirror  # noqa: E402

NB = 3 * 4096 * 14336 * 2


def main():
    m = HostMirror(4 * NB)
    dst = torch.empty(4 * NB, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    out = {}
    for nstreams in (1, 2, 4):
        for chunks in (1, 4, 16):
            for _ in range(2):  # warm + measured
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for rep in range(4):
                    per = NB // chunks
                    for c in range(chunks):
                        s = streams[(rep * chunks + c) % nstreams]
                        s.wait_event(a)
                        N.call("bm_memcpy", dst.data_ptr() + rep * NB + c * per, m.ptr + rep * NB + c * per, per,
                               s.cuda_stream)
                for s in streams[:nstreams]:
                    ev = torch.cuda.Event()
                    ev.record(s)
                    torch.cuda.current_stream().wait_event(ev)
                b.record()
                torch.cuda.synchronize()
            out[f"streams{nstreams}_chunks{chunks}"] = 4 * NB / (a.elapsed_time(b) / 1e3) / 1e9
    print(json.dumps({"bytes_per_expert": NB, "h2d_gbs": out, "best": max(out.values())}))
    m.close()


if __name__ == "__main__":
    main()
