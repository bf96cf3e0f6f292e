#!/bin/bash
set -u
bash tools/ncu_nvlink.sh 2 1 . gpu__time_duration.sum _all
bash tools/ncu_nvlink.sh 2 1 fused "" _fused
