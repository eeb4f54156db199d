#!/bin/bash
# One GPU session's evidence: GPU tests, the bench line, the ncu launch list of the bench command and one
# `ncu --set full` capture of the iteration kernels.  Usage (on the B200 box, from the repo root):
#   bash tools/gpu_round.sh <tag> [tests|bench|ncu]...   (default: all three)
set -u
tag=${1:-r02}; shift || true
what=${*:-tests bench ncu}
mkdir -p gpurun_out
for w in $what; do
  case $w in
    tests)
      timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${tag}_gputests.log 2>&1
      echo "tests rc=$?" >> gpurun_out/${tag}_rc.log ;;
    check)
      DABA_LIB=$PWD/paper_2305_07026_b200/libdaba_check.so timeout 2400 python -m pytest tests/test_gpu_parity.py \
        tests/test_gpu_bal.py tests/test_gpu_coarse.py -q --timeout 900 -p no:cacheprovider \
        > gpurun_out/${tag}_check_tests.log 2>&1
      echo "check rc=$?" >> gpurun_out/${tag}_rc.log ;;
    bench)
      python bench.py --steps 100 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
      echo "bench rc=$?" >> gpurun_out/${tag}_rc.log ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
        > gpurun_out/${tag}_ncu_launches.log 2>&1
      echo "ncu-launches rc=$?" >> gpurun_out/${tag}_rc.log
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cam_pass|k_pt_sum|k_cam_solve" \
        -c 3 -o gpurun_out/${tag}_full -f python tools/prof_run.py --iters 2 > gpurun_out/${tag}_ncu_full.log 2>&1
      echo "ncu-full rc=$?" >> gpurun_out/${tag}_rc.log ;;
  esac
done
cat gpurun_out/${tag}_rc.log
