#!/bin/bash
# ncu --set full of every preprocessing kernel (router + linear branch) of one cfg2 forward
ncu --set full --import-source on --clock-control none -k regex:"colmean|pool_project|project_kernel|kprep|router_rows|kphi_htot|lin_reduce" \
    -c 8 -o gpurun_out/ncu_prep_cfg2 -f python tools/profile_forward.py --config cfg2 > gpurun_out/ncu_prep.log 2>&1
