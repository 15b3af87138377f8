"""Debug: one SD-1.5 ragged step (3 requests) + decode, print ok / error."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
from paper_2605_08835_b200.engine import Engine
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
hw = int(sys.argv[2]) if len(sys.argv) > 2 else 64
eng = Engine("sd15", max_latent_hw=hw, b_max=4, precision=prec)
eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
slots = [eng.register(torch.from_numpy(synth.text_embedding(1, i, 77, 768))) for i in range(3)]
lat = [torch.from_numpy(synth.initial_noise(1, i, hw, hw)).cuda() for i in range(3)]
eng.step(lat, [0, 20, 45], [50] * 3, [1, 0, 1], [7.5, 7.5, 4.0], slots)
torch.cuda.synchronize()
print("step ok", prec, hw, float(lat[0].abs().mean()))
