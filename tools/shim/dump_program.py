"""Writes a BASELINE HDMR config's program as a flat binary file for
tools/shim/bench_shim.cpp (the C++-shim timing of a reference-style caller).

Format (little endian): int32 d, m, n_slots; f64 f_anchor[m]; per slot:
int32 order, int32 dims[order], int32 b, int32 mode, int32 max_level,
f64 eps_gamma, int64 n_nodes, uint32 keys[n_nodes][order], f64 surplus[n_nodes][m].
Usage: python tools/shim/dump_program.py <config> <out.bin>
"""
import struct
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np

from paper_2202_06555_b200 import workloads as W


def main():
    cid, out = int(sys.argv[1]), sys.argv[2]
    cfg = W.CONFIGS[cid]
    parts = W.build_hdmr_parts(cfg)
    with open(out, "wb") as f:
        f.write(struct.pack("<iii", cfg.d, cfg.m, len(parts.slots)))
        f.write(np.ascontiguousarray(parts.f_anchor, dtype="<f8").tobytes())
        for u, b, g in parts.slots:
            f.write(struct.pack("<i", len(u)))
            f.write(np.array(u, dtype="<i4").tobytes())
            if g is None:
                f.write(struct.pack("<iiidq", b, 1, 1, 0.0, 0))
                continue
            keys, sur = g.nodes()
            f.write(struct.pack("<iiidq", b, g.boundary_mode, g.max_level, g.eps_gamma, keys.shape[0]))
            f.write(np.ascontiguousarray(keys, dtype="<u4").tobytes())
            f.write(np.ascontiguousarray(sur, dtype="<f8").tobytes())
    print(out, len(parts.slots), "slots")


if __name__ == "__main__":
    main()
