#!/bin/bash
# tests + bench + ncu launch list + full capture (one gpurun call)
bash tools/gpu_check.sh
bash tools/profile.sh
