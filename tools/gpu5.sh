GS_LIB_PATH=build_variants/lib_prof512.so timeout 300 python tools/profile_run.py cfg3
GS_LIB_PATH=build_variants/lib_c8t512s8.so timeout 300 python tools/profile_run.py cfg3
