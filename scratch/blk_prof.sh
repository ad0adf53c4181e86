BDEM_LIB=/root/repo/scratch/lib_blocked.so BDEM_ROW_ORDER=strip python scratch/shfl_micro.py > gpurun_out/blk_plain.log 2>&1 && \
BDEM_LIB=/root/repo/scratch/lib_blocked.so BDEM_ROW_ORDER=strip ncu --set full --clock-control none -k regex:"k_spmv$" -s 5 -c 1 -o gpurun_out/prof_blk -f python scratch/shfl_micro.py > gpurun_out/ncu_blk.log 2>&1
BDEM_ROW_ORDER=strip ncu --set full --clock-control none -k regex:"k_spmv$" -s 5 -c 1 -o gpurun_out/prof_strided_strip -f python scratch/shfl_micro.py > gpurun_out/ncu_ss.log 2>&1
python profiles/summarize.py gpurun_out/prof_blk.ncu-rep gpurun_out/prof_strided_strip.ncu-rep > gpurun_out/blk_summary.txt
