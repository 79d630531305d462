# Round 2 first GPU pass: fused cov/corr parity + timing, GPU suite, smoke, default bench.
set -x
mkdir -p gpurun_out
bash scripts/gram_run.sh > gpurun_out/r2a_gram.log 2>&1
tail -40 gpurun_out/r2a_gram.log
TAG=r2a bash scripts/round_quick.sh
