"""Fixed fit launch for ncu captures of the encoder kernel (never a bench number)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402
from paper_2306_16699_b200 import encoder as E, synth  # noqa: E402
from transforms_common import smooth_images  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 296
x = torch.from_numpy(smooth_images(n, 32, 32, seed=1)).cuda()
dm = E.init_batch(synth.ARCH_A, range(n), 32, 32)
for _ in range(3):
    E.train_batch(dm, x, 5e-4, 50)
torch.cuda.synchronize()
print("ok")
