"""Sweep HostTextParser's chunk size (cfg2-schema text, 1M lines).

Run on the GPU box: python tools/parse_chunk_sweep.py
Prints lines/s per chunk size: mean of 5 synchronous calls after 1 warm-up."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2407_10115_b200.features import HostTextParser, InputSchema, split_lines  # noqa: E402


def main():
    n = 1_000_000
    names, lines = bench.make_text_lines(n)
    sc = InputSchema(tuple(names), frozenset(names[20:]), 24)
    buf, off = split_lines(("\n".join(lines) + "\n").encode())
    h_text = torch.from_numpy(buf.copy()).pin_memory()
    h_off = torch.from_numpy(off).pin_memory()
    h_status = torch.empty(n, dtype=torch.int32).pin_memory()
    dev = torch.device("cuda", 0)
    for chunk in (1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18):
        p = HostTextParser(sc, dev, n, len(buf), chunk_lines=chunk)
        p(h_text, h_off, h_status)
        assert int((h_status != 0).sum()) == 0
        t0 = time.perf_counter()
        for _ in range(5):
            p(h_text, h_off, h_status)
        dt = (time.perf_counter() - t0) / 5
        print(f"chunk={chunk:>7}: {n / dt / 1e6:6.1f} M lines/s", flush=True)
        del p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
