import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import sigkern_oracle as O
from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian, sig_kernel_gram
for (nx, ny, lx, ly, d, M) in [(2, 2, 300, 300, 2, 3), (3, 2, 600, 300, 2, 3), (2, 2, 2048, 2048, 4, 8), (5, 4, 520, 520, 3, 4)]:
    X = gen_brownian(nx, lx, d, SeedStream(1)).data; Y = gen_brownian(ny, ly, d, SeedStream(2)).data
    cfg = KernelConfig(n_levels=M)
    K = sig_kernel_gram(X, Y, cfg=cfg); K64 = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
    print(nx, ny, lx, ly, d, M, "maxrel", float(np.max(np.abs(K - K64) / np.abs(K64))))
