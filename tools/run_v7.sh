bash tools/gpu_ab.sh librs.so librs_A_MINB_6.so librs_A_MINB_7.so librs_A_MINB_8.so librs.so
ABX="--config lj" bash tools/gpu_ab.sh librs.so librs_A_MINB_6.so librs_A_MINB_7.so
