"""Scenario runner and trajectory evaluation at GPU scale.

Mirrors the reference's end-to-end harness:
* ``run_scenario``   — sim/scenario.cpp:303-392 (world -> sampled map -> engine,
  per frame: simulated scan -> make_scan_cloud -> FilterEngine::step, stats.csv,
  snapshots, est/gt TUM files, report.txt). The scan of each frame goes
  through the device pipeline (``FilterEngine.step_points``: make_scan_cloud on
  the GPU, bit-identical to the host path).
* ``evaluate_ate`` / ``format_report`` — eval.cpp:32-116 (translation ATE,
  convergence frame = first frame of a run of ``conv_sustain`` frames under
  both thresholds, recovery frames after each occlusion window).
* ``write_tum`` / ``read_tum`` / ``write_odometry`` / ``read_odometry`` —
  trajectory_io.cpp:10-92.
* ``localization_config`` — the acceptance suite's corridor calibration
  (acceptance.cpp:275-289), used for criteria C6 (global localization) and C7
  (kidnap recovery) at 1e5..1e6 particles.
"""
import math
import os

import numpy as np

from . import sim
from .abi import make_config
from .api import FilterEngine


class AteOptions:
    def __init__(self, align=False, conv_trans=1.0, conv_rot_deg=10.0, conv_sustain=10, occlusions=()):
        self.align, self.conv_trans, self.conv_rot_deg = align, conv_trans, conv_rot_deg
        self.conv_sustain, self.occlusions = conv_sustain, list(occlusions)


class EvalReport:
    def __init__(self):
        self.n_frames, self.skip = 0, 0
        self.ate_rmse = self.ate_mean = self.ate_std = self.ate_max = 0.0
        self.convergence_frame = -1
        self.ate_rmse_post_convergence = -1.0
        self.recovery_frames = []
        self.mean_times = {}

    def as_dict(self):
        return dict(self.__dict__)


def rotation_angle_between(a, b):
    """se3.hpp:152-155."""
    Ra, Rb = np.asarray(a[:9]).reshape(3, 3), np.asarray(b[:9]).reshape(3, 3)
    c = 0.5 * (np.trace(Ra.T @ Rb) - 1.0)
    return math.acos(min(1.0, max(-1.0, c)))


def _first_sustained(terr, rerr_deg, start, opts):
    """eval.cpp:13-27."""
    run = 0
    for i in range(max(start, 0), len(terr)):
        if terr[i] < opts.conv_trans and rerr_deg[i] < opts.conv_rot_deg:
            run += 1
            if run >= opts.conv_sustain:
                return i - opts.conv_sustain + 1
        else:
            run = 0
    return -1


def _umeyama(src, dst):
    """Eigen::umeyama(src, dst, false): rigid transform (no scaling) of 3xN columns."""
    mu_s, mu_d = src.mean(1, keepdims=True), dst.mean(1, keepdims=True)
    cov = (dst - mu_d) @ (src - mu_s).T / src.shape[1]
    U, _, Vt = np.linalg.svd(cov)
    S = np.eye(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        S[2, 2] = -1.0
    R = U @ S @ Vt
    return R, (mu_d - R @ mu_s).reshape(3)


def evaluate_ate(estimated, truth, skip=0, opts=None):
    """eval.cpp:32-94. estimated / truth: sequences of (stamp, pose12)."""
    opts = opts or AteOptions()
    if len(estimated) != len(truth):
        raise ValueError("evaluate_ate: trajectory length mismatch")
    n = len(estimated)
    rep = EvalReport()
    rep.n_frames, rep.skip = n, skip
    if n == 0:
        return rep
    Rc, tc = np.eye(3), np.zeros(3)
    if opts.align:
        src = np.stack([np.asarray(e[1])[9:] for e in estimated], 1)
        dst = np.stack([np.asarray(t[1])[9:] for t in truth], 1)
        Rc, tc = _umeyama(src, dst)
    terr, rerr = np.zeros(n), np.zeros(n)
    for i in range(n):
        e, t = np.asarray(estimated[i][1], float), np.asarray(truth[i][1], float)
        est = sim.pose_of(Rc @ e[:9].reshape(3, 3), Rc @ e[9:] + tc)
        terr[i] = np.linalg.norm(est[9:] - t[9:])
        rerr[i] = rotation_angle_between(est, t) * 180.0 / math.pi
    sel = terr[max(skip, 0):]
    if len(sel):
        rep.ate_mean = float(sel.sum() / len(sel))
        rep.ate_rmse = float(math.sqrt((sel * sel).sum() / len(sel)))
        rep.ate_std = float(math.sqrt(max(0.0, (sel * sel).sum() / len(sel) - rep.ate_mean ** 2)))
        rep.ate_max = float(sel.max())
    rep.convergence_frame = _first_sustained(terr, rerr, skip, opts)
    if rep.convergence_frame >= 0:
        post = terr[rep.convergence_frame:]
        rep.ate_rmse_post_convergence = float(math.sqrt((post * post).sum() / len(post)))
    for (_, end) in opts.occlusions:
        r = _first_sustained(terr, rerr, end, opts)
        rep.recovery_frames.append(r - end if r >= 0 else -1)
    rep.terr, rep.rerr_deg = terr, rerr
    return rep


def format_report(rep):
    """eval.cpp:96-114."""
    out = [f"frames: {rep.n_frames}", f"skip: {rep.skip}", f"ate_rmse: {rep.ate_rmse:.6f}",
           f"ate_mean: {rep.ate_mean:.6f}", f"ate_std: {rep.ate_std:.6f}", f"ate_max: {rep.ate_max:.6f}",
           f"convergence_frame: {rep.convergence_frame}",
           f"ate_rmse_post_convergence: {rep.ate_rmse_post_convergence:.6f}"]
    out += [f"recovery_frames_{w}: {r}" for w, r in enumerate(rep.recovery_frames)]
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------- trajectory I/O (trajectory_io.cpp)
def quat_of_R(R):
    """Eigen::Quaterniond(Matrix3d) (trace / max-diagonal branches) -> (x, y, z, w)."""
    R = np.asarray(R, float).reshape(3, 3)
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        t = math.sqrt(tr + 1.0)
        w = 0.5 * t
        t = 0.5 / t
        return ((R[2, 1] - R[1, 2]) * t, (R[0, 2] - R[2, 0]) * t, (R[1, 0] - R[0, 1]) * t, w)
    i = 0
    if R[1, 1] > R[0, 0]:
        i = 1
    if R[2, 2] > R[i, i]:
        i = 2
    j, k = (i + 1) % 3, (i + 2) % 3
    t = math.sqrt(R[i, i] - R[j, j] - R[k, k] + 1.0)
    q = [0.0, 0.0, 0.0]
    q[i] = 0.5 * t
    t = 0.5 / t
    w = (R[k, j] - R[j, k]) * t
    q[j] = (R[j, i] + R[i, j]) * t
    q[k] = (R[k, i] + R[i, k]) * t
    return (q[0], q[1], q[2], w)


def R_of_quat(qx, qy, qz, qw):
    """pose_from_quat (trajectory_io.cpp:10-17): normalised quaternion -> rotation."""
    n = math.sqrt(qx * qx + qy * qy + qz * qz + qw * qw)
    x, y, z, w = qx / n, qy / n, qz / n, qw / n
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def write_tum(path, traj):
    with open(path, "w") as f:
        for stamp, p in traj:
            p = np.asarray(p, float)
            qx, qy, qz, qw = quat_of_R(p[:9])
            f.write(f"{stamp:.6f} {p[9]:.9f} {p[10]:.9f} {p[11]:.9f} {qx:.9f} {qy:.9f} {qz:.9f} {qw:.9f}\n")


def read_tum(path):
    traj = []
    with open(path) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            v = [float(x) for x in line.split()]
            if len(v) < 8:
                raise RuntimeError(f"read_tum: malformed line in {path}")
            traj.append((v[0], sim.pose_of(R_of_quat(v[4], v[5], v[6], v[7]), np.array(v[1:4]))))
    return traj


def write_odometry(path, odo):
    with open(path, "w") as f:
        for delta, cov, valid in odo:
            d = np.asarray(delta, float)
            qx, qy, qz, qw = quat_of_R(d[:9])
            c = np.asarray(cov, float).reshape(6, 6)
            vals = [d[9], d[10], d[11], qx, qy, qz, qw] + [c[r, k] for r in range(6) for k in range(r, 6)]
            f.write(" ".join(f"{v:.12g}" for v in vals) + f" {1 if valid else 0}\n")


def read_odometry(path):
    out = []
    with open(path) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            v = line.split()
            if len(v) < 7 + 21 + 1:
                raise RuntimeError(f"read_odometry: malformed line in {path}")
            x = [float(t) for t in v[:28]]
            cov = np.zeros((6, 6))
            it = iter(x[7:28])
            for r in range(6):
                for k in range(r, 6):
                    cov[r, k] = cov[k, r] = next(it)
            out.append((sim.pose_of(R_of_quat(*x[3:7]), np.array(x[:3])), cov.reshape(36), int(v[28]) != 0))
    return out


def write_snapshot(path, particles):
    """scenario.cpp:289-299: id, t, quaternion, log_post per particle."""
    with open(path, "w") as f:
        for i in range(particles.n):
            p = particles.poses[i]
            qx, qy, qz, qw = quat_of_R(p[:9])
            f.write(f"{particles.id[i]} {p[9]:.9f} {p[10]:.9f} {p[11]:.9f} {qx:.9f} {qy:.9f} {qz:.9f} {qw:.9f} "
                    f"{particles.log_post[i]:.9g}\n")


# ---------------------------------------------------------------- scenario runs
def localization_config(seed, n_particles=100000, **kw):
    """acceptance.cpp:275-289 (desk-scale corridor calibration)."""
    return make_config(n_particles=n_particles, seed=seed, nnf_resolution=0.1, full_rotation=1, sigma_r=50.0,
                       sigma_t=25.0, repulsion_gain=0.005, lsh_alpha=0.016, beta=5.0, miss_cost=50.0,
                       gn_scan_stride=2, **kw)


class ScenarioResult:
    def __init__(self):
        self.truth, self.estimated, self.frames = [], [], []
        self.report = None


def run_scenario(sc, cfg, out_dir="", snapshot_every=0, device=0, n_frames=None):
    """scenario.cpp:303-392 on one B200 (scans prepared on the device)."""
    writing = bool(out_dir)
    if writing:
        os.makedirs(out_dir, exist_ok=True)
        if snapshot_every > 0:
            os.makedirs(os.path.join(out_dir, "snapshots"), exist_ok=True)
    rects, mapc = sim.scenario_map(sc, cfg)
    eng = FilterEngine(mapc, cfg, device=device)
    eng.init_uniform(mapc.bounds)
    nf = sc.n_frames if n_frames is None else min(n_frames, sc.n_frames)
    truth_poses = sim.build_trajectory(sc)[:nf]
    odo = sim.build_odometry(sc, truth_poses)
    dt = 1.0 / sc.rate_hz
    res = ScenarioResult()
    res.truth = [(f * dt, p) for f, p in enumerate(truth_poses)]
    stats = open(os.path.join(out_dir, "stats.csv"), "w") if writing else None
    if stats:
        stats.write("frame,stamp,occluded,rep_id,rep_x,rep_y,rep_z,rep_log_post,trans_err,mean_n_matched,"
                    "observation_rejected,overflow,predict_ms,neighbor_ms,likelihood_ms,update_ms,posterior_ms,"
                    "total_ms\n")
    keys = ["predict_ms", "neighbor_ms", "likelihood_ms", "update_ms", "posterior_ms", "total_ms"]
    sums = {k: 0.0 for k in keys}
    for f in range(nf):
        pts = sim.scan_points_for_frame(sc, rects, truth_poses, f)
        d, c, v = odo[f]
        fr = eng.step_points(pts, d, c, v)
        res.frames.append(fr)
        res.estimated.append((f * dt, fr["representative"]))
        for k in keys:
            sums[k] += fr[k]
        if stats:
            rp = fr["representative"]
            terr = float(np.linalg.norm(rp[9:] - truth_poses[f][9:]))
            stats.write(f"{f},{f * dt:.3f},{fr['scan_empty']},{fr['rep_id']},{rp[9]:.6f},{rp[10]:.6f},{rp[11]:.6f},"
                        f"{fr['rep_log_post']:.6g},{terr:.6f},{fr['mean_n_matched']:.2f},"
                        f"{fr['observation_rejected']},{fr['neighbor_stats']['overflow_dropped']},"
                        + ",".join(f"{fr[k]:.3f}" for k in keys) + "\n")
        if writing and snapshot_every > 0 and f % snapshot_every == 0:
            write_snapshot(os.path.join(out_dir, "snapshots", f"snap_{f:06d}.txt"), eng.particles())
    if stats:
        stats.close()
    occl = [(b, e) for b, e in sc.occlusions if e <= nf]
    res.report = evaluate_ate(res.estimated, res.truth, 0, AteOptions(occlusions=occl))
    res.report.mean_times = {k: sums[k] / max(nf, 1) for k in keys}
    if writing:
        write_tum(os.path.join(out_dir, "est.tum"), res.estimated)
        write_tum(os.path.join(out_dir, "gt.tum"), res.truth)
        with open(os.path.join(out_dir, "report.txt"), "w") as fh:
            fh.write(f"scenario: {sc.name}\nseed: {sc.seed}\nparticles: {cfg.n_particles}\n")
            fh.write(format_report(res.report))
    eng.close()
    return res
