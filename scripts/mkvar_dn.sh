# mkvar_dn.sh NAME "FLAGS": builds build_probe/libbl_NAME.so with decoder_net.cu compiled with FLAGS
set -e
cd /root/repo/paper_2101_05600_b200/csrc
JSON_INC=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$JSON_INC $2 -c decoder_net.cu -o /root/repo/build_probe/dn_$1.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared build/decode_m0.o build/decode_m1.o build/decode_m2.o build/decode_m3.o build/decode_m4.o build/capi.o build/gemm_tcgen05.o build/encoder.o /root/repo/build_probe/dn_$1.o -o /root/repo/build_probe/libbl_$1.so
