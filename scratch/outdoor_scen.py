import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2404_16370_b200 import scenario as S, sim
for n, sensor_az in ((1 << 20, 256),):
    sc = sim.scenario_preset("outdoor_kidnap", seed=7)
    sc.sensor = sim.sensor_spec(n_azimuth=sensor_az, elevations_deg=list(np.linspace(-30.0, 30.0, 8)), max_range=60.0)
    for variant, kw in (("default", {}), ("loc", "loc")):
        if kw == "loc":
            cfg = S.localization_config(11, n_particles=n)
            cfg.nnf_resolution = 0.2
            cfg.nnf_max_query_dist = 2.0
        else:
            from paper_2404_16370_b200.abi import make_config
            cfg = make_config(n_particles=n, seed=11, nnf_resolution=0.2, nnf_max_query_dist=2.0)
        cfg.n_scan_max = 512
        t = time.time()
        res = S.run_scenario(sc, cfg)
        r = res.report
        terr = r.terr
        print(variant, n, f"conv={r.convergence_frame} post_ate={r.ate_rmse_post_convergence:.3f} recovery={r.recovery_frames} "
              f"mean_ms={r.mean_times['total_ms']:.2f} wall={time.time()-t:.1f}s")
        print("  terr every 10:", np.round(terr[::10], 2).tolist())
