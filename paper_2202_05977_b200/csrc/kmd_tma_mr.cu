// kmd_tma_mr.cu -- the TMA kernel of kmd_tma.cu compiled with 28-row tiles
// (namespace tma28) for the "Ours MR" levels (NEXT row 2; PAPER.md:313-318,
// Eq. 7): every 2 x 2 block of a level lies in one tile, so the level's Eq. 7
// combine with the next-coarser level runs in the tile's epilogue and the
// fine level's filtered image never goes to HBM.  Its layout is fixed here
// (build-variant switches of kmd_tma.cu do not apply to this translation unit).
#undef KMD_SEG
#undef KMD_NB
#undef KMD_NV
#undef KMD_VS
#undef KMD_BBW
#undef KMD_NFIELD
#undef KMD_VSPLIT
#undef KMD_HFUSE
#undef KMD_STAGGER
#define KMD_TH 28
#define KMD_NB 3  // 28-row boxes: a 4-deep blend ring does not fit beside the 4-deep V ring
#define KMD_TMA_NS tma28
#define KMD_TMA_SECONDARY 1
#include "kmd_tma.cu"
