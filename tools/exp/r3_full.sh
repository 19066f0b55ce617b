timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputests_r03.txt
cat gpurun_out/gputests_r03.txt
bash tools/exp/r3_sanitize.sh
