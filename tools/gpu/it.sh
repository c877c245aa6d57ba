NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --nvtx --nvtx-include "iter/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/it_c1.csv python tools/prof_iter.py --config 1 > gpurun_out/it_c1.log 2>&1; echo it=$?; tail -2 gpurun_out/it_c1.log
