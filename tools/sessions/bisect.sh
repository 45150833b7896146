for c in "38 3 1 70" "36 3 1 70" "37 3 1 70" "100 3 1 70" "120 3 1 70" "130 3 1 70" "250 3 1 70" "37 3 1 70 host" "138 3 1 70"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/bisect_case.py $c 2>&1 | grep -E "^case|Error" | tail -1
done
