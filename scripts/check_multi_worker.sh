mkdir -p gpurun_out/mw
python tests/multi_gpu_worker.py gpurun_out/mw 1 && python -c "
import numpy as np; d=np.load('gpurun_out/mw/rank0.npz'); print(d.files, d['fits'])"
python -m pytest tests/test_gpu_multi.py -q -rs 2>&1 | tail -3
