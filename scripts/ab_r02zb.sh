python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)
import ctypes; cr=ctypes.CDLL('libcudart.so.12') if False else None
" > gpurun_out/l2info.txt 2>&1
python - >> gpurun_out/l2info.txt 2>&1 <<'PY'
from cuda.bindings import runtime as rt
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0); print("max persisting L2", err, v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0); print("max window", err, v)
PY
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "p64|PSFS_X=1|--l2-persist 67108864" "p96|PSFS_X=1|--l2-persist 100663296" "p32|PSFS_X=1|--l2-persist 33554432"
done > gpurun_out/ab_r02zb.txt 2>&1
