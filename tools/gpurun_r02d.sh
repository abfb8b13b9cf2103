mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ssp tools/slice_stream_probe.cu
( for t in 0 1; do
  echo "test_wait=$t cfg4 RS4 NS16"; /tmp/ssp 131072 29344 4 16 1 $t | head -2
  echo "test_wait=$t cfg4 RS2 NS32"; /tmp/ssp 131072 29344 2 32 1 $t | head -2
  echo "test_wait=$t cfg5 RS1 NS18"; /tmp/ssp 65536 104512 1 18 1 $t | head -2
  echo "test_wait=$t cfg5 RS2 NS9"; /tmp/ssp 65536 104512 2 9 1 $t | head -2
  done ) > gpurun_out/ssp.txt 2>&1
