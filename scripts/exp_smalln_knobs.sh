#!/bin/bash
# smalln pipeline experiments: band-ring depth (variant libs) x poll back-off, with/without band+MMA work
L=$GRAFT_REPO_ROOT/paper_2602_06071_b200
mkdir -p gpurun_out
CFG=${CFG:-smalln} TAG=${TAG:-e4} ENVS="base:X=1 sleep0:BPS_TC_SLEEP=0 nb5:BPS_LIB=$L/libbps_nb5.so nb5s0:BPS_LIB=$L/libbps_nb5.so,BPS_TC_SLEEP=0 nb8:BPS_LIB=$L/libbps_nb8.so nb8s0:BPS_LIB=$L/libbps_nb8.so,BPS_TC_SLEEP=0 ls_s0:BPS_TC_SLEEP=0" bash scripts/ab_env.sh
