"""One ragged denoising step and a 2-chunk VAE decode through the C ABI, for compute-sanitizer runs
(memcheck / racecheck / synccheck) of the tcgen05 / TMA / mbarrier pipelines:

  SD_NO_GRAPH=1 compute-sanitizer --tool racecheck python tools/sanitize_step.py sd15 16 fp16
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "tiny"
hw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prec = sys.argv[3] if len(sys.argv) > 3 else "fp16"
eng = Engine(model, max_latent_hw=hw, b_max=4, c_max=2, precision=prec)
L, D = eng.ctx_len, eng.ctx_dim
pu = torch.from_numpy(synth.uncond_pooled(0, eng.pooled_dim)) if eng.pooled_dim else None
eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, L, D)), pu)
slots = [eng.register(torch.from_numpy(synth.text_embedding(1, i, L, D)),
                      torch.from_numpy(synth.pooled_embedding(1, i, eng.pooled_dim)) if eng.pooled_dim else None)
         for i in range(3)]
lat = [torch.from_numpy(synth.initial_noise(1, i, hw, hw)).cuda() for i in range(3)]
eng.step(lat, [0, 20, 45], [50] * 3, [1, 0, 1], [7.5, 7.5, 4.0], slots)
img = eng.decode(lat[0], 2)
torch.cuda.synchronize()
assert np.isfinite(img.cpu().numpy()).all() and np.isfinite(lat[1].cpu().numpy()).all()
print("sanitize step ok", model, hw, prec, flush=True)
eng.close()
