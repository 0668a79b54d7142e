"""Write bench_data/c3_observations.npz: the C3 observations (SURVEY §8(d):
trivariate n_s=1675, n_t=48, n_r=1, 80 400 per process, seed 2) produced by
the package's generator (synthetic.generate_synthetic, the reference's draw
order; pinned to the reference's input checksums by
tests/test_gpu_baseline_configs.py).  bench.py's reference arm rebuilds the
designs with the reference's own build_spec (the first draws of the same
seeded generator) and reads these observations, so the CPU reference f_obj
runs on the same model without the CPU latent draw (one C3 POBTAF)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic  # noqa: E402

TRUE = [-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00, 0.00, 0.60, -0.40,
        0.30]

if __name__ == "__main__":
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), TRUE, seed=2,
                              device=torch.device("cuda", 0))
    os.makedirs(os.path.join(ROOT, "bench_data"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "bench_data", "c3_observations.npz"),
                        **{f"y{i}": np.asarray(y) for i, y in enumerate(data.spec.observations)})
    print("written", [float(np.sum(y)) for y in data.spec.observations])
