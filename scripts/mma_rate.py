"""Cycles per 16-wide K step of the bf16x6 product shapes (tcprobe.cu fdsdf_probe_mma_rate)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_08980_b200 import fdsdf

L = fdsdf.lib()
L.fdsdf_probe_mma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
out = torch.zeros(1, dtype=torch.int64, device="cuda")
names = {0: "1-range 6 x N", 1: "3-range 3N,2N,N", 2: "2-range 2N,2N,N,N", 3: "single N"}
for n in (32, 48, 64, 80):
    for mode in (3, 0, 1, 2):
        if mode == 1 and 3 * n > 256:
            continue
        iters = 400
        assert L.fdsdf_probe_mma_rate(mode, n, iters, out.data_ptr()) == 0
        assert L.fdsdf_probe_mma_rate(mode, n, iters, out.data_ptr()) == 0
        cyc = out.item() / (iters * 4)
        nsum = {0: 6 * n, 1: 6 * n, 2: 6 * n, 3: n}[mode]
        floor = 128 * nsum / 256
        print(f"N={n:3d} {names[mode]:20s} {cyc:7.1f} cyc/kstep  floor {floor:6.1f}  ratio {cyc / floor:4.2f}")

# TMEM load throughput (tcprobe.cu fdsdf_probe_tmem_rate)
L.fdsdf_probe_tmem_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
sink = torch.zeros(1, device="cuda")
for width in (8, 16):
    for nw in (4, 8, 16):
        iters = 2000
        assert L.fdsdf_probe_tmem_rate(width, nw, iters, out.data_ptr(), sink.data_ptr()) == 0
        assert L.fdsdf_probe_tmem_rate(width, nw, iters, out.data_ptr(), sink.data_ptr()) == 0
        cyc = out.item()
        byts = nw * iters * 32 * width * 4
        print(f"tcgen05.ld x{width:2d} {nw:2d} warps: {byts / cyc:6.1f} B/cycle  ({cyc / iters:6.1f} cyc per warp-load round)")

# CTA pair (cta_group::2, M = 256): cycles per K step for the whole pair
L.fdsdf_probe_mma_rate2.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
names2 = {0: "6 x N", 1: "3 x 3N (9 products)", 2: "2N,2N,N,N", 3: "single N"}
for n in (64, 80):
    for mode in (3, 0, 2, 1):
        if mode == 1 and 3 * n > 256:
            continue
        iters = 400
        assert L.fdsdf_probe_mma_rate2(mode, n, iters, out.data_ptr()) == 0
        assert L.fdsdf_probe_mma_rate2(mode, n, iters, out.data_ptr()) == 0
        cyc = out.item() / (iters * 4)
        print(f"pair N={n:3d} {names2[mode]:22s} {cyc:7.1f} cyc/kstep (M=256)  = {cyc / 2:6.1f} per M=128 half")
