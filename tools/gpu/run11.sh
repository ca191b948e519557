timeout 900 python -m pytest tests -m gpu -x -q -k "pretrain_public or sprm or prepass" > gpurun_out/r2_gputest11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest11.log
tail -4 gpurun_out/r2_gputest11.log
./tools/x2/ntchain
