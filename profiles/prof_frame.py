"""Profiling driver (run under ncu; never a bench number): one configs[2]
frame (camera 0) or one configs[3] training view, after warm-up frames that
size the workspaces.

  python profiles/prof_frame.py render [frames]   # preprocess, bin, raster
  python profiles/prof_frame.py train [views]     # + loss, K6, K7
"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2509_07021_b200 import scenes  # noqa: E402
from paper_2509_07021_b200.loss import image_loss  # noqa: E402
from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer  # noqa: E402
from paper_2509_07021_b200.render import LossConfig  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "render"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    rast = Rasterizer()
    if mode == "render":
        scene, cams = scenes.config2(n_cams=1)
        g = GaussianTensors.from_arrays(scene)
        for _ in range(reps):
            rast.forward(g, cams[0], check=True, track=False)
    else:
        scene, cams = scenes.config3()
        g = GaussianTensors.from_arrays(scene)
        tgt = torch.from_numpy(scenes.target_image(0, cams[0].height, cams[0].width)).cuda()
        for _ in range(reps):
            fr = rast.forward(g, cams[0], check=True)
            _, dimg, _ = image_loss(fr.img, tgt, LossConfig(), grad="f32")
            rast.backward(g, fr, dimg, mask_grads=True)
    torch.cuda.synchronize()
    print("done", mode, reps)


if __name__ == "__main__":
    main()
