cd tools/micro
for t in 8192 16384 26624; do for st in 2 3 4; do for c in 1 2 3 4; do ./tma_ring $t $st $c 400; done; done; done
