import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_zeropoint import _one_signed
from oracle import rinr_oracle as O
from paper_2306_16699_b200 import synth, Store
mb, sh = _one_signed(synth.ARCH_A, 4, 7, 1.0)
mb2, _ = _one_signed(synth.ARCH_C, 4, 7, 1.0)
for mbx, size in ((mb, 8), (mb2, 8)):
    data = synth.archive_bytes(mbx)
    models = O.read_models(data)
    want = np.stack(O.decode_batch(models, size, size))
    with Store(data) as st:
        p = st.dequantize(torch.arange(4)).cpu().numpy()
        print("dq", all(np.array_equal(p[i, :O.flat_params(m).size], O.flat_params(m)) for i, m in enumerate(models)))
        got = st.decode(torch.arange(4), size, size, layout="nhwc", precision="exact", sin="accurate").cpu().numpy()
        print(np.abs(got - want).max())
        print(got[0, :2, :4, 0]); print(want[0, :2, :4, 0])
        print(st.info.hidden_int8 if hasattr(st.info, 'hidden_int8') else '')
