import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2407_19097_b200.neural import UNet, UNetConfig, init_params
import oracle
cfg = UNetConfig(input_channels=4)
params = init_params(cfg)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
H, W = int(sys.argv[1]), int(sys.argv[2])
x = torch.rand((H, W, 4), device=dev, generator=g)
tc = UNet(cfg, params, device=dev)(x)
tc2 = UNet(cfg, params, device=dev)(x)
os.environ["NAR_UNET_SIMT"] = "1"
simt = UNet(cfg, params, device=dev)(x)
d = (tc - simt).double()
print(H, W, "tc-vs-simt psnr", 10*np.log10(1/float((d**2).mean())), "max", float(d.abs().max()), "tc repeat identical:", bool(torch.equal(tc, tc2)))
if H * W <= 256 * 512:
    ref = oracle.forward(x.cpu().numpy()[None], params, cfg)[0]
    print("tc-vs-oracle psnr", oracle.psnr(tc.cpu().numpy(), ref), "simt-vs-oracle", oracle.psnr(simt.cpu().numpy(), ref))
