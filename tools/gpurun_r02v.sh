mkdir -p gpurun_out
for c in 4 2 8 16 32; do echo "chunks $c" >> gpurun_out/v_obuild.txt; IRL_OBUILD_CHUNKS=$c timeout 300 python tools/obuild_time.py 3,4,5 >> gpurun_out/v_obuild.txt 2>&1; done
