// temporary: head entry points land in dpt.cu / seg.cu / det.cu
#include "util.cuh"
extern "C" {
int vpe_dpt_create(const vpe_dpt_config*, const vpe_dpt_weights*, vpe_dpt**) { return VPE_E_CONFIG; }
int vpe_dpt_destroy(vpe_dpt*) { return VPE_OK; }
int vpe_dpt_forward(vpe_dpt*, const void* const*, float*, float*, void*) { return VPE_E_CONFIG; }
int vpe_seg_create(const vpe_seg_config*, const vpe_seg_weights*, vpe_seg**) { return VPE_E_CONFIG; }
int vpe_seg_destroy(vpe_seg*) { return VPE_OK; }
int vpe_seg_forward(vpe_seg*, const void*, uint8_t*, float*, void*) { return VPE_E_CONFIG; }
int vpe_det_create(const vpe_det_config*, const vpe_det_weights*, vpe_det**) { return VPE_E_CONFIG; }
int vpe_det_destroy(vpe_det*) { return VPE_OK; }
int vpe_det_forward(vpe_det*, const void*, const vpe_det_outputs*, void*) { return VPE_E_CONFIG; }
}
