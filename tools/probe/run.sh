cd "$(dirname "$0")"
for cfg in "16 16 0 0" "36 18 0 0" "36 18 -1 -1" "32 16 0 0" "16 8 -1 0" "16 8 0 -1"; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -DBOXX=$1 -DBOXY=$2 -DCX=$3 -DCY=$4 -o /tmp/tp tma_probe.cu -lcuda 2>&1 | tail -2
  /tmp/tp | tail -2
done
