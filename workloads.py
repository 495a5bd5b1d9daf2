"""The five BASELINE.json configurations (+ the SURVEY NEXT-3 Black-Scholes workload) as plain
data (no arithmetic of the method).

Shared by tests/ and bench.py; neither the oracle nor the product imports it.
"""
from dataclasses import dataclass, replace
from typing import Optional, Tuple


@dataclass(frozen=True)
class Workload:
    name: str
    problem: str          # "heat" | "hjb" | "allen_cahn" | "black_scholes"
    d: int
    w: int
    N: int
    T: float
    batch: int            # global paths per iteration
    precision: str        # "fp32" | "bf16"
    lr: float
    iterations: int
    seed: int = 0
    levels: Optional[Tuple[int, ...]] = None     # multilevel grids (config 4)
    iters_per_level: int = 0
    x0: float = 0.0       # X_0 = x0 * ones(d)
    formulation: str = "per_step"   # "per_step" (north_star) | "shared" (the paper's own, NEXT-1)
    arch: str = "fc"      # shared: "fc" | "resnet"
    layers: int = 2       # shared: tanh layers of width w

    def with_(self, **kw):
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: heat BSDE, closed form u(0,0) = 2dT = 20
    "cfg1_heat": Workload("cfg1_heat", "heat", 10, 20, 5, 1.0, 256, "fp32", 1e-2, 200),
    # configs[1]: HJB / LQ control, Cole-Hopf check
    "cfg2_hjb": Workload("cfg2_hjb", "hjb", 100, 110, 20, 1.0, 16384, "fp32", 1e-2, 2000),
    # configs[2]: Allen-Cahn, bf16 operands / fp32 accumulate
    "cfg3_allen_cahn": Workload("cfg3_allen_cahn", "allen_cahn", 100, 110, 20, 0.3, 65536,
                                "bf16", 5e-4, 4000),
    # configs[3]: multilevel HJB, N = 5 -> 80, fixed budget per level (400)
    "cfg4_hjb_multilevel": Workload("cfg4_hjb_multilevel", "hjb", 100, 110, 5, 1.0, 65536,
                                    "fp32", 1e-2, 2000, levels=(5, 10, 20, 40, 80),
                                    iters_per_level=400),
    # configs[4]: scale-out Allen-Cahn, 524288 paths sharded over 1/2/4/8 GPUs
    "cfg5_allen_cahn_scaleout": Workload("cfg5_allen_cahn_scaleout", "allen_cahn", 100, 110, 80,
                                         0.3, 524288, "bf16", 5e-4, 1000),
    # Black-Scholes d = 100, r = 0.05, σ = 0.4; T, N, x0
    # and the batch are not given by the paper: T = 1, N = 20, B = 65536 as config 3, and
    # x0 = 0.1 so that u(0, x0) = e^{0.21}·d·0.01 ≈ 1.234 (DESIGN R21)
    "nx3_black_scholes": Workload("nx3_black_scholes", "black_scholes", 100, 110, 20, 1.0, 65536,
                                  "bf16", 1e-2, 2000, x0=0.1),
    # the paper's own formulation on its Table 1 workload (P:299, P:319,
    # P:488): Black-Scholes d = 100, M = 100 paths, N = 50 steps, one network of 4 tanh
    # layers x 256 shared by all steps, Adam lr 1e-3, 20 000 iterations, fp32
    "nx1_shared_bs_paper": Workload("nx1_shared_bs_paper", "black_scholes", 100, 256, 50, 1.0, 100,
                                    "fp32", 1e-3, 20000, x0=0.1, formulation="shared", layers=4),
    # the paper's ResNet and NAIS-Net rows of the same table (R23, R26)
    "nx1_shared_bs_resnet_paper": Workload("nx1_shared_bs_resnet_paper", "black_scholes", 100, 256,
                                           50, 1.0, 100, "fp32", 1e-3, 20000, x0=0.1,
                                           formulation="shared", arch="resnet", layers=4),
    "nx2_shared_bs_nais_paper": Workload("nx2_shared_bs_nais_paper", "black_scholes", 100, 256, 50,
                                         1.0, 100, "fp32", 1e-3, 20000, x0=0.1,
                                         formulation="shared", arch="nais", layers=4),
    # the same with bf16 tcgen05 row GEMMs (weight gradients fp32)
    "nx1_shared_bs_paper_bf16": Workload("nx1_shared_bs_paper_bf16", "black_scholes", 100, 256, 50,
                                         1.0, 100, "bf16", 1e-3, 20000, x0=0.1,
                                         formulation="shared", layers=4),
    "nx1_shared_bs_m4096_bf16": Workload("nx1_shared_bs_m4096_bf16", "black_scholes", 100, 256, 50,
                                         1.0, 4096, "bf16", 1e-3, 20000, x0=0.1,
                                         formulation="shared", layers=4),
    # the same network and problem at a throughput batch (M = 4096)
    "nx1_shared_bs_m4096": Workload("nx1_shared_bs_m4096", "black_scholes", 100, 256, 50, 1.0, 4096,
                                    "fp32", 1e-3, 20000, x0=0.1, formulation="shared", layers=4),
}
