nvidia-smi; nproc; lscpu | grep -E "Model name|^CPU\(s\)|Flags" | cut -c1-400
python -c "import numpy as np; np.show_runtime()" 2>&1 | head -40
python - <<'PY'
import numpy as np
rng=np.random.default_rng(0)
re=rng.standard_normal(200000)*np.exp2(rng.integers(-60,60,200000)); im=re*np.exp2(rng.uniform(-30,30,200000))*np.sign(rng.standard_normal(200000))
c=re+1j*im
a=np.abs(c)
big=np.maximum(np.abs(re),np.abs(im)); small=np.minimum(np.abs(re),np.abs(im))
r=np.where(big==0,0,small/big)
import math
f=np.array([math.sqrt(math.fma(x,x,1.0)) if hasattr(math,'fma') else 0 for x in r[:10]])
print("has fma", hasattr(math,'fma'))
print("eq naive", np.mean(a==np.sqrt(re*re+im*im)))
PY
