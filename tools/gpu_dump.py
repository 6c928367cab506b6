"""Run the CUDA path on small scenes and dump raw segments + images to
gpurun_out/dump_<name>.npz for offline comparison with the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import scenegen as sg  # noqa: E402
from parity_util import gpu_run  # noqa: E402

SCENES = {
    "shell1": lambda: sg.shell_uniform(1, 48, 8, gl_points=6),
    "shell2": lambda: sg.shell_uniform(2, 64, 16, gl_points=6),
    "shell3": lambda: sg.shell_uniform(3, 96, 16, gl_points=6),
}

if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    for name in (sys.argv[1:] or SCENES):
        g = gpu_run(SCENES[name]())
        np.savez_compressed(f"gpurun_out/dump_{name}.npz", raw=g["raw"], rgba=g["rgba"], hpp=g["hits_per_pixel"],
                            visible=g["visible"], nf=g["newton_failures"], ff=g["face_failures"])
        print(name, g["count"], g["hit_pairs"], g["newton_failures"], g["face_failures"])
