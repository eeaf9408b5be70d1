"""Shared-memory bank model of the fused FFT twiddle lookups under candidate paddings."""
from collections import defaultdict
def wavefronts(addrs):  # addrs: float2 indices for 32 lanes; 2 half-warps
    tot=0
    for h in range(2):
        banks=defaultdict(set)
        for a in addrs[16*h:16*h+16]:
            banks[(2*a)%32].add(a); banks[(2*a+1)%32].add(a)
        tot+=max(len(v) for v in banks.values())
    return tot
pads={'none':lambda m:m,'m+m>>3':lambda m:m+(m>>3),'m+m>>4':lambda m:m+(m>>4),'m+m>>2':lambda m:m+(m>>2),'m+m>>5':lambda m:m+(m>>5),
      'xor':lambda m: m ^ ((m>>4)&15), 'xor3':lambda m: m ^ ((m>>5)&15), 'm+m>>3+m>>6': lambda m: m+(m>>3)+(m>>6), 'xor_lo':lambda m: m ^ ((m>>3)&7)}
# pass2 pattern: t1024[pad(j*k)], j=1..31, k=lane (0..31)
for name,f in pads.items():
    t=sum(wavefronts([f(j*k) for k in range(32)]) for j in range(1,32))
    # tlo pattern in pass3: m = 4*j*k (k = column index, varies by lane: k = tid + 512c -> lane), tlo[m & 255]
    t2=sum(wavefronts([f((4*j*k)&255) for k in range(32)]) for j in range(1,16))
    print(f"{name:14s} pass2 {t:4d} (ideal {2*31})  tlo {t2:4d} (ideal {2*15})")
