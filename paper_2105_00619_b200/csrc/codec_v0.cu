// codec_v0.cu -- the exact64 variant's kernels and entry points
// (see codec_impl.cuh).
#include "codec_impl.cuh"

namespace optb_b200 {

cudaError_t encode_v0(const Geom& g, const RowSrc& rs, bool vec, void* cont, uint8_t* offs, cudaStream_t s, int sms,
                       uint64_t* launches) {
  if (vec) return enc_vec<0>(g, rs, cont, offs, s, sms, launches);
  return enc_generic<0>(g, rs, cont, offs, s, sms, launches);
}

cudaError_t decode_v0(const Geom& g, const void* cont, const uint8_t* offs, const Epi& e, bool vec, void* out,
                       DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  if (vec) return dec_vec_any<0>(g, cont, offs, e, out, err, s, sms, launches);
  return dec_generic_any<0>(g, cont, offs, e, out, err, s, sms, launches);
}

cudaError_t roundtrip_v0(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs,
                          const Epi& e, void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  return rt_vec_any<0>(cm, g, rs, cont, offs, e, out, err, s, sms, launches);
}

}  // namespace optb_b200
