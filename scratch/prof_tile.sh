set -e
mkdir -p gpurun_out
python scratch/roworder_ab.py z > gpurun_out/tile_plain.txt 2>&1
ncu --set full --clock-control none -k regex:k_spmv_tile -s 3 -c 1 -o gpurun_out/tile_full -f python scratch/roworder_ab.py z > gpurun_out/tile_ncu.log 2>&1
ncu -i gpurun_out/tile_full.ncu-rep --page raw --csv > gpurun_out/tile_full_raw.csv
