"""Extract numpy's ziggurat tables (ki_double, wi_double, fi_double) from the
installed libnpyrandom.a and emit csrc/ziggurat_tables.h; verify a pure-Python
model of Generator(Philox).standard_normal against numpy bit for bit.

numpy's standard_normal (numpy/random/src/distributions/distributions.c,
random_standard_normal): r = next_uint64; idx = r & 0xff; r >>= 8; sign = r & 1;
rabs = (r >> 1) & (2^52-1); x = rabs * wi[idx] (negated if sign); accept if
rabs < ki[idx]; else idx == 0 -> tail loop with log1p, otherwise wedge test
with exp.  Philox4x64-10 keyed (seed, stream), counter pre-incremented.
"""
import math
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "paper_2310_09417_b200", "csrc", "ziggurat_tables.h")


def extract():
    lib = os.path.join(os.path.dirname(np.__file__), "random", "lib", "libnpyrandom.a")
    d = tempfile.mkdtemp()
    subprocess.run(["ar", "x", lib], cwd=d, check=True)
    obj = os.path.join(d, "src_distributions_distributions.c.o")
    subprocess.run(["objcopy", "-O", "binary", "--only-section=.rodata", obj, os.path.join(d, "ro.bin")], check=True)
    ro = open(os.path.join(d, "ro.bin"), "rb").read()
    syms = {}
    for line in subprocess.run(["objdump", "-t", obj], capture_output=True, text=True).stdout.splitlines():
        parts = line.split()
        if parts and parts[-1] in ("ki_double", "wi_double", "fi_double") and ".rodata" in line:
            syms[parts[-1]] = int(parts[0], 16)
    ki = struct.unpack("<256Q", ro[syms["ki_double"]:syms["ki_double"] + 2048])
    wi = struct.unpack("<256d", ro[syms["wi_double"]:syms["wi_double"] + 2048])
    fi = struct.unpack("<256d", ro[syms["fi_double"]:syms["fi_double"] + 2048])
    return ki, wi, fi


M64 = (1 << 64) - 1
R = 3.6541528853610088
INV_R = 0.27366123732975828


class PhiloxModel:
    def __init__(self, seed, stream):
        self.key = [seed & M64, stream & M64]
        self.ctr = [0, 0, 0, 0]
        self.buf = []

    def _block(self):
        c = self.ctr
        for i in range(4):  # pre-increment the 256-bit counter
            c[i] = (c[i] + 1) & M64
            if c[i] != 0:
                break
        x = list(c)
        k0, k1 = self.key
        for _ in range(10):
            p0 = 0xD2E7470EE14C6C93 * x[0]
            p1 = 0xCA5A826395121157 * x[2]
            hi0, lo0 = p0 >> 64, p0 & M64
            hi1, lo1 = p1 >> 64, p1 & M64
            x = [hi1 ^ x[1] ^ k0, lo1, hi0 ^ x[3] ^ k1, lo0]
            k0 = (k0 + 0x9E3779B97F4A7C15) & M64
            k1 = (k1 + 0xBB67AE8584CAA73B) & M64
        self.buf = x

    def next64(self):
        if not self.buf:
            self._block()
        return self.buf.pop(0)

    def next_double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def normal(g, ki, wi, fi):
    while True:
        r = g.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            return x
        if idx == 0:
            while True:
                xx = -INV_R * math.log1p(-g.next_double())
                yy = -math.log1p(-g.next_double())
                if yy + yy > xx * xx:
                    return -(R + xx) if ((rabs >> 8) & 1) else R + xx
        else:
            if (fi[idx - 1] - fi[idx]) * g.next_double() + fi[idx] < math.exp(-0.5 * x * x):
                return x


def main():
    ki, wi, fi = extract()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
    for seed, stream in ((0, 0), (3, 77), (0, 0x123456789ABCDEF)):
        g = PhiloxModel(seed, stream)
        ours = np.array([normal(g, ki, wi, fi) for _ in range(n)])
        ref = np.random.Generator(np.random.Philox(key=[seed, stream])).standard_normal(n)
        assert np.array_equal(ours.view(np.uint64), ref.view(np.uint64)), (seed, stream)
    with open(OUT, "w") as f:
        f.write("// numpy Generator.standard_normal ziggurat tables (ki_double, wi_double,\n")
        f.write("// fi_double), extracted from the installed libnpyrandom.a by\n")
        f.write("// tools/gen_ziggurat_tables.py and verified bitwise against numpy.\n#pragma once\n#include <stdint.h>\n\n")
        f.write("namespace rs {\n")
        f.write("__device__ __constant__ uint64_t zig_ki[256] = {\n")
        f.write(",\n".join("  0x%016xull" % v for v in ki) + "};\n")
        for name, arr in (("zig_wi", wi), ("zig_fi", fi)):
            bits = [struct.unpack("<Q", struct.pack("<d", v))[0] for v in arr]
            f.write(f"__device__ __constant__ uint64_t {name}_bits[256] = {{\n")
            f.write(",\n".join("  0x%016xull" % v for v in bits) + "};\n")
        f.write("}  // namespace rs\n")
    print(f"tables verified on {3 * n} normals; wrote {OUT}")


if __name__ == "__main__":
    main()
