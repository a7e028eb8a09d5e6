"""Small instances of every CUDA kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck; one tool per gpurun call):

    compute-sanitizer --tool memcheck --kernel-name regex:'rinr|decode|prep|fit|ser_' python tools/sanitize_cases.py

decode_persist (narrow net: separable and general layer 0, fp32 / bf16,
accurate sine, crop), decode_tc (wide net, fp32 / bf16), decode_generic,
dequantize, prune_l1 / quantize / psnr, the GPU writer and the encoder fit."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16699_b200 import Store, encoder, synth, transforms as T  # noqa: E402
from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD, resized_crop_params  # noqa: E402


def main():
    a = synth.gpu_store_bytes("c2", 64, seed=1)
    c = synth.gpu_store_bytes("c3", 3, seed=1)
    with Store(a) as st:
        ids = torch.arange(16, device="cuda")
        st.dequantize(ids)
        st.decode(ids, 32, 32, precision="fp32")                      # separable layer 0
        st.decode(ids, 32, 32, precision="bf16", dtype=torch.bfloat16)
        st.decode(ids, 24, 40, precision="fp32", layout="nhwc")         # general layer 0
        st.decode(ids, 13, 7, precision="fp32", sin="accurate")
        st.decode(ids, 13, 7, precision="exact")                        # decode_generic
        st.decode(ids, 32, 32, aug=resized_crop_params(16), aug_mode="crop", mean=IMAGENET_MEAN, std=IMAGENET_STD)
    with Store(c) as st:
        ids = torch.arange(3, device="cuda")
        for prec in ("fp32", "bf16"):
            st.decode(ids, 40, 40, precision=prec, aug=resized_crop_params(3), aug_mode="crop", mean=IMAGENET_MEAN,
                      std=IMAGENET_STD, dtype=torch.bfloat16)
    mb = synth.tweak_r1(synth.random_batch(synth.ARCH_A, 8, 3))
    dm = T.DeviceModels.from_batch(mb)
    T.prune_l1(dm, 0.2)
    q = T.quantize(dm, "affine8")
    T.serialize(dm, q)
    T.psnr(torch.rand(4, 8, 8, 3, device="cuda"), torch.rand(4, 8, 8, 3, device="cuda"))
    imgs = torch.rand(2, 16, 16, 3, device="cuda")
    fit = encoder.init_batch(synth.ARCH_A, [1, 2], 16, 16)
    encoder.train_batch(fit, imgs, 5e-4, 4)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
