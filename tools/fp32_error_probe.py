"""FP32 MC path vs FP64 on identical streams: per-path F_T and price errors
(the distribution behind tests/test_gpu_mc.py's FP32 tolerances)."""
import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2407_20713_b200 as pkg
import os, ctypes
lib=os.environ.get('SABR_LIB')
eng=pkg.Engine(0, lib=ctypes.CDLL(lib)) if lib else pkg.Engine(0)
F0,T=2257.37,0.495890
for params in [pkg.StaticSabrParams(0.375162, 0.999999, 0.331441, -0.999999), pkg.StaticSabrParams(0.3, 0.7, 0.5, -0.4), pkg.CaseIParams(0.393329, 1.0, -1.0, 0.941565, 0.001, 1.246906)]:
  for rng in ['xoshiro','philox']:
    p64=pkg.SimulationPlan(num_paths=1<<16, seed=9, rng=rng); p32=pkg.SimulationPlan(num_paths=1<<16, seed=9, rng=rng); p32.precision='fp32'
    a=eng.simulate_terminals(params,F0,params.alpha,T,p64); b=eng.simulate_terminals(params,F0,params.alpha,T,p32)
    e=np.abs(a-b)/a
    x=eng.price_european_batch(params,F0,[0.9*F0,F0,1.1*F0],0.018196,0.034516,T,p64)
    y=eng.price_european_batch(params,F0,[0.9*F0,F0,1.1*F0],0.018196,0.034516,T,p32)
    pe=max(abs(u.value-v.value)/max(u.value,1e-300) for u,v in zip(x,y) if u.value > 0)
    print(type(params).__name__, rng, 'path err p50 %.2e p99 %.2e p99.99 %.2e max %.2e  worst at %d' % (np.median(e), np.percentile(e,99), np.percentile(e,99.99), e.max(), e.argmax()), 'price err %.2e' % pe)
