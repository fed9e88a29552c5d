nproc; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"; lscpu | grep -E 'Model name|Socket|Thread|Core'; free -g | head -2
nvidia-smi; nvidia-smi topo -m
python - <<'PY'
import torch
p=torch.cuda.get_device_properties(0)
print(p)
print('L2', p.L2_cache_size, 'SMs', p.multi_processor_count)
PY
