# configs[4] max elements per GPU: the Helmholtz per_shape_P table at 100 GB per cell, final kernels
timeout 2400 python bench.py --sweep on --sweep-quick --sweep-gb 100 --sweep-tables helm_deformed --steps 5 > gpurun_out/r2run72_maxsweep.json 2> gpurun_out/r2run72_maxsweep.err; echo "maxsweep rc=$?"
tail -c 300 gpurun_out/r2run72_maxsweep.err
