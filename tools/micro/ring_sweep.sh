# TMA bulk-copy ring bandwidth (tools/micro/tma_ring.cu): tile bytes x stages x CTAs/SM
cd "$(dirname "$0")"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -cudart shared -o /tmp/tma_ring tma_ring.cu || exit 1
for cfg in "26624 2 3" "26624 8 1" "26624 6 1" "24576 4 2" "26624 3 2" "16384 6 2" "16384 4 3" "12288 8 2" "8192 8 3" "20480 5 2"; do
  /tmp/tma_ring $cfg 400
done
