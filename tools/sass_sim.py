"""Rough issue model of a SASS loop body (CPU-side tuning aid, not a profiler).

usage: python tools/sass_sim.py SASS_FILE START_HEX END_HEX [--warps W] [--steps S] [--iters N]

Parses the instructions in [START, END) of a `cuobjdump -sass` listing with
their control words, then replays the body N times for W warps sharing one SM
sub-partition (SMSP), one instruction issued per cycle:
  * fixed-latency dependencies follow the compiler's own stall counts
    (control bits 41-44: the warp waits that many cycles after issuing);
  * variable-latency results (LDS, LDG, SHFL, ...) set a scoreboard (bits 46-48
    write barrier, 49-51 read barrier) and consumers wait on its mask (52-57);
    the barrier clears after LAT cycles (LDS ~30, SHFL 24 measured);
  * fp64 instructions occupy the SMSP's fp64 pipe for 2 cycles (16 lanes).
Memory waits on the cp.async groups (DEPBAR) and global loads are modelled as
satisfied, so the result is a lower bound: cycles per step per SMSP.
"""
import re
import sys

LAT = {"LDS": 30, "SHFL": 24, "LDL": 40, "LDG": 500, "S2R": 20, "LDSM": 30, "LDGSTS": 20, "STS": 4,
       "STG": 4, "STL": 4, "BAR": 20}
FP64 = {"DADD", "DMUL", "DFMA", "DSETP"}
MIO = {"LDS", "STS", "SHFL", "LDSM"}

ins_re = re.compile(r"/\*([0-9a-f]+)\*/\s+(@!?U?P[0-9T]\s+)?([A-Z0-9_.]+)\s*([^;]*);\s*/\*\s*0x([0-9a-f]+)\s*\*/")
hi_re = re.compile(r"^\s*/\*\s*0x([0-9a-f]+)\s*\*/\s*$")


def parse(path, lo, hi):
    lines = open(path).read().splitlines()
    out = []
    for n, line in enumerate(lines):
        m = ins_re.search(line)
        if not m:
            continue
        addr = int(m.group(1), 16)
        if addr < lo or addr >= hi:
            continue
        h = hi_re.match(lines[n + 1])
        ctl = int(h.group(1), 16) if h else 0
        stall = (ctl >> 41) & 0xF
        wbar = (ctl >> 46) & 0x7
        rbar = (ctl >> 49) & 0x7
        wmask = (ctl >> 52) & 0x3F
        base = m.group(3).split(".")[0]
        out.append((base, stall, wbar, rbar, wmask))
    return out


def simulate(body, warps=2, iters=3):
    n = len(body)
    pc = [0] * warps
    next_ok = [0] * warps  # earliest issue cycle (stall counts)
    sb = [[0] * 6 for _ in range(warps)]  # scoreboard release cycles
    fp64_free = 0
    mio_free = 0
    cyc = 0
    done = [0] * warps
    total = n * iters
    last = 0
    while min(done) < total:
        for k in range(warps):
            w = (last + 1 + k) % warps
            if done[w] >= total or next_ok[w] > cyc:
                continue
            base, stall, wbar, rbar, wmask = body[pc[w]]
            if any((wmask >> b) & 1 and sb[w][b] > cyc for b in range(6)):
                continue
            if base in FP64 and fp64_free > cyc:
                continue
            if base in MIO and mio_free > cyc:
                continue
            if wbar != 7:
                sb[w][wbar] = cyc + LAT.get(base, 20)
            if rbar != 7:
                sb[w][rbar] = max(sb[w][rbar], cyc + 4)
            if base in FP64:
                fp64_free = cyc + 2
            if base in MIO:
                mio_free = cyc + 1
            next_ok[w] = cyc + max(1, stall)
            pc[w] = (pc[w] + 1) % n
            done[w] += 1
            last = w
            break
        cyc += 1
    return cyc


if __name__ == "__main__":
    path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
    warps = int(sys.argv[sys.argv.index("--warps") + 1]) if "--warps" in sys.argv else 2
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 3
    body = parse(path, lo, hi)
    nfp = sum(1 for b in body if b[0] in FP64)
    cyc = simulate(body, warps, iters)
    per = cyc / iters / steps
    print(f"{len(body)} instructions ({nfp} fp64) per body, {warps} warps/SMSP: {cyc} cycles for {iters} bodies"
          f" -> {per:.0f} cycles per step per SMSP ({per / warps:.0f} per warp-step),"
          f" fp64 pipe {2 * nfp * iters * warps / cyc:.2f}")
