#!/bin/bash
bash tools/gpu_check.sh
bash tools/ab/run_ab.sh $1
