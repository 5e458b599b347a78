import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from helpers import config, cube_set, room_scene
from paper_2404_16370_b200.api import FilterEngine
rects, mapc, scan = room_scene()
parts = cube_set(3000, 7, 20)
e = FilterEngine(mapc, config(nnf_resolution=0.2, likelihood_mode=2))
e.set_particles(parts)
ll, nm = e.evaluate_likelihoods(scan)
np.save(sys.argv[1], np.concatenate([ll, nm.astype(np.float64)]))
