make -j16 BUILD=build_dbg LIB=ablibs/dbg.so NVFLAGS_EXTRA=-DKNN_WS2_DEBUG ablibs/dbg.so > /dev/null 2>&1 || echo buildfail
KNN_LIB_PATH=ablibs/dbg.so python scripts/dbg_sel2.py 2>&1 | head -30
