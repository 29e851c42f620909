import numpy as np, sys
for m in ["d","s","sd"]:
    a=np.load("gpurun_out/u_asym_%s.npy"%m); b=np.load("gpurun_out/u_sym_%s.npy"%m)
    print(m, "sym vs asym rel L2 %.3e"%(np.linalg.norm(a-b)/np.linalg.norm(a)))
