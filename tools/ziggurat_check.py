"""(CPU) numpy's standard_normal restated on the ziggurat tables read out of
libnpyrandom.a (tools/gen_ziggurat.py) and the Philox model (oracle/philox.py):
bit-identical values and final generator state over N draws.
Usage: python tools/ziggurat_check.py [N]"""
import math, sys, time
import os
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, 'tools'))
import numpy as np
from oracle.philox import PhiloxModel
import gen_ziggurat
t = gen_ziggurat.tables()
KI, WI, FI = t['ki_double'], t['wi_double'], t['fi_double']
R = 3.6541528853610088
INV_R = 0.27366123732975828
def next_double(ph): return (ph.next64() >> 11) * (1.0 / 9007199254740992.0)
def std_normal(ph):
    while True:
        r = ph.next64()
        idx = r & 0xff
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000fffffffffffff
        x = rabs * WI[idx]
        if sign: x = -x
        if rabs < KI[idx]: return x
        if idx == 0:
            while True:
                xx = -INV_R * math.log1p(-next_double(ph))
                yy = -math.log1p(-next_double(ph))
                if yy + yy > xx * xx:
                    return -(R + xx) if ((rabs >> 8) & 1) else R + xx
        else:
            if (FI[idx - 1] - FI[idx]) * next_double(ph) + FI[idx] < math.exp(-0.5 * x * x):
                return x
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
g = np.random.Generator(np.random.Philox(123))
ph = PhiloxModel(g.bit_generator.state)
t0 = time.time()
want = g.standard_normal(n)
got = np.array([std_normal(ph) for _ in range(n)])
print("equal:", np.array_equal(got.view(np.int64), want.view(np.int64)), "tails(|x|>3.654):", int((np.abs(want) > R).sum()), time.time() - t0)
st = g.bit_generator.state
print("state equal:", [int(x) for x in st['state']['counter']] == ph.ctr, st['buffer_pos'] == ph.pos)
